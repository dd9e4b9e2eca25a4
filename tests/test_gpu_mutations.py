"""The parity suite's own sensitivity, on the GPU (SURVEY §8(c) "sabotage env var", S:522;
VERDICT r1 "a deliberately injected skip-one-store mutation fails").

The mutations live only in the testing build (libhydra_test.so, -DHYDRA_TESTING); the
release library has no such switches (tests/test_capi_cpu.py).  Each case runs in a
subprocess that loads the testing build (HYDRA_TESTING=1), calls the library through
tests/nanfill.py exactly as the parity tests do, and reports whether the parity gate
caught the mutation:
  combine_bug        Eq. 5 combine without its rescaling (w_p = 1)
  skip_prefix_store  persistent tcgen05 prefix kernel: CTA 0 skips one 4-row store group
  skip_pair_store    CTA-pair prefix kernel: worker 0 skips the stores of 4 rows
  skip_suffix_store  tensor-core suffix kernel: CTA 0 skips head 0's row of its first item
  skip_short_store   short-suffix kernel (suffix_short.cu): the same skipped row
  clean              no mutation: the same calls must pass (control)
Also: the testing build's device check of the lens precondition counts lens[b] > S_cap and
lens[b] < 0 (hydra_debug_lens_violations)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
import numpy as np, torch
import oracle, synth
import paper_2402_05099_b200 as hydra
from tests import nanfill as H
from tests.util import assert_parity, problem_to

assert hydra.get_config("testing_build") == 1, hydra.version()
DEV = "cuda:0"
res = {}

def run(case):
    for k in ("prefix_impl", "suffix_impl", "inject_combine_bug", "mutate"):
        hydra.set_config(k, 0)
    hydra.set_config("prefix_variant", 6)
    if case in ("combine_bug", "clean_composite"):
        if case == "combine_bug":
            hydra.set_config("inject_combine_bug", 1)
        pb = synth.make_problem(8, 8, 2, 128, 500, 60, dtype="bf16", dist="mixed", seed=12)
        t = problem_to(pb, DEV)
        out, lse = H.hydragen_attention(t["q"], t["pk"], t["pv"], t["sk"], t["sv"], t["lens"], return_lse=True)
        ref, lref = oracle.flat_attention(pb)
    elif case in ("skip_prefix_store", "clean_prefix", "skip_pair_store", "clean_pair"):
        hydra.set_config("prefix_impl", 3)
        hydra.set_config("prefix_variant", 9 if "pair" in case else 6)
        if case == "skip_prefix_store":
            hydra.set_config("mutate", 1)
        if case == "skip_pair_store":
            hydra.set_config("mutate", 3)
        pb = synth.make_problem(300, 8, 2, 128, 1100, 1, dtype="bf16", dist="mixed", seed=4)
        t = problem_to(pb, DEV)
        out, lse = H.prefix_attn(t["q"], t["pk"], t["pv"])
        ref, lref = oracle.prefix_only(pb)
    elif case in ("clean_short", "skip_short_store"):
        hydra.set_config("suffix_impl", 3)
        if case == "skip_short_store":
            hydra.set_config("mutate", 2)
        pb = synth.make_problem(40, 8, 2, 128, 0, 200, dtype="bf16", dist="mixed", seed=7)
        t = problem_to(pb, DEV)
        out, lse = H.suffix_attn(t["q"], t["sk"], t["sv"], t["lens"])
        ref, lref = oracle.suffix_only(pb)
    else:
        hydra.set_config("suffix_impl", 2)
        if case == "skip_suffix_store":
            hydra.set_config("mutate", 2)
        pb = synth.make_problem(40, 8, 2, 128, 0, 300, dtype="bf16", dist="mixed", seed=6)
        t = problem_to(pb, DEV)
        out, lse = H.suffix_attn(t["q"], t["sk"], t["sv"], t["lens"])
        ref, lref = oracle.suffix_only(pb)
    torch.cuda.synchronize()
    try:
        assert_parity(out, ref, lse, lref, what=case)
        return "pass"
    except AssertionError as e:
        return "caught: " + str(e)[:80]

for case in ("clean_composite", "combine_bug", "clean_prefix", "skip_prefix_store", "clean_pair", "skip_pair_store",
             "clean_suffix", "skip_suffix_store", "clean_short", "skip_short_store"):
    res[case] = run(case)

# lens precondition: device check in the testing build
for k in ("prefix_impl", "suffix_impl", "inject_combine_bug", "mutate"):
    hydra.set_config(k, 0)
pb = synth.make_problem(4, 8, 2, 128, 100, 32, lens=[32, 0, 5, 32], dtype="bf16", dist="mixed", seed=3)
t = problem_to(pb, DEV)
hydra._lib.load().hydra_debug_lens_violations(1)
t["lens"].copy_(torch.tensor([40, -3, 5, 32], dtype=torch.int32))
H.hydragen_attention(t["q"], t["pk"], t["pv"], t["sk"], t["sv"], t["lens"])
res["lens_violations"] = int(hydra._lib.load().hydra_debug_lens_violations(1))
print("RESULT " + json.dumps(res))
"""


@pytest.fixture(scope="module")
def results():
    env = dict(os.environ, HYDRA_TESTING="1", PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-c", SCRIPT], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=600)
    line = [x for x in r.stdout.splitlines() if x.startswith("RESULT ")]
    assert r.returncode == 0 and line, r.stdout[-2000:] + r.stderr[-3000:]
    return json.loads(line[0][7:])


@pytest.mark.parametrize("case", ["clean_composite", "clean_prefix", "clean_pair", "clean_suffix", "clean_short"])
def test_unmutated_testing_build_passes(results, case):
    assert results[case] == "pass", results[case]


@pytest.mark.parametrize("case", ["combine_bug", "skip_prefix_store", "skip_pair_store", "skip_suffix_store",
                                  "skip_short_store"])
def test_mutation_is_caught(results, case):
    assert results[case].startswith("caught"), f"{case} passed the parity gate"


def test_lens_precondition_counted(results):
    assert results["lens_violations"] == 2  # lens 40 > S_cap 32 and lens -3 < 0
