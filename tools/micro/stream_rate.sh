# per-SM streaming rate by load path (see stream_rate.cu)
for m in ${MODES:-0 1 2 3 4 5 6 7}; do for c in ${CTAS:-16 64 148}; do for st in ${STAGES:-2 4 6}; do
  if [ $m = 3 ] && [ $st != 2 ]; then continue; fi
  timeout 30 tools/micro/stream_rate $m $c $st; done; done; done
