"""Decode-loop integration: the KV
append kernel, and attention + append replayed from one CUDA graph with device-side
lengths, checked against the fp64 oracle at every step."""
import dataclasses

import numpy as np
import pytest
import torch

import oracle
import synth
from tests import nanfill as H
from tests.util import assert_parity, problem_to

hydra = pytest.importorskip("paper_2402_05099_b200")

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


def _bits(t: torch.Tensor) -> np.ndarray:
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def test_append_kv_exact():
    """Rows land at position lens[b] bit-exactly, nothing else changes, full caches are left alone."""
    B, Hkv, d, S = 5, 2, 128, 10
    pb = synth.make_problem(B, 4, Hkv, d, 0, S, lens=[0, 3, 9, 10, 5], dtype="bf16", seed=3)
    t = problem_to(pb, DEV)
    g = torch.Generator(device=DEV).manual_seed(0)
    k_new = torch.randn(B, Hkv, d, device=DEV, generator=g).bfloat16()
    v_new = torch.randn(B, Hkv, d, device=DEV, generator=g).bfloat16()
    sk0, sv0 = _bits(t["sk"]), _bits(t["sv"])
    hydra.append_kv(k_new, v_new, t["sk"], t["sv"], t["lens"])
    torch.cuda.synchronize()
    sk1, sv1, lens1 = _bits(t["sk"]), _bits(t["sv"]), t["lens"].cpu().numpy()
    kb, vb = _bits(k_new), _bits(v_new)
    for b, L in enumerate([0, 3, 9, 10, 5]):
        if L < S:
            assert lens1[b] == L + 1
            assert (sk1[b, L] == kb[b]).all() and (sv1[b, L] == vb[b]).all()
            keep = [s for s in range(S) if s != L]
            assert (sk1[b, keep] == sk0[b, keep]).all() and (sv1[b, keep] == sv0[b, keep]).all()
        else:  # full cache: unchanged
            assert lens1[b] == S and (sk1[b] == sk0[b]).all() and (sv1[b] == sv0[b]).all()


def test_append_kv_rejects_bad_arguments():
    k = torch.zeros(2, 2, 128, dtype=torch.bfloat16, device=DEV)
    sk = torch.zeros(2, 4, 2, 128, dtype=torch.bfloat16, device=DEV)
    lens = torch.zeros(2, dtype=torch.int32, device=DEV)
    with pytest.raises(ValueError):
        hydra.append_kv(k[:, :1], k[:, :1], sk, sk, lens)  # wrong head count
    with pytest.raises(TypeError):
        hydra.append_kv(k.float(), k.float(), sk, sk, lens)  # dtype mismatch


@pytest.mark.parametrize("aux", [False, True])
def test_decode_loop_in_one_graph(aux):
    """Each replay: append this step's token K/V (inputs copied into static buffers), then
    attend over prefix + the grown suffixes.  Step t's output must match the oracle over
    the caches as they are after step t's append (App. B attention)."""
    B, Hq, Hkv, d, P, S = 6, 8, 2, 128, 300, 40
    lens0 = np.array([0, 5, 17, 1, 30, 12], np.int32)
    pb = synth.make_problem(B, Hq, Hkv, d, P, S, lens=lens0, dtype="bf16", dist="mixed", seed=41)
    t = problem_to(pb, DEV)
    steps = 4
    gk = torch.Generator(device=DEV).manual_seed(1)
    new_k = [torch.randn(B, Hkv, d, device=DEV, generator=gk).bfloat16() for _ in range(steps)]
    new_v = [torch.randn(B, Hkv, d, device=DEV, generator=gk).bfloat16() for _ in range(steps)]
    k_in = torch.empty(B, Hkv, d, dtype=torch.bfloat16, device=DEV)
    v_in = torch.empty_like(k_in)
    out = torch.empty(B, Hq, d, dtype=torch.bfloat16, device=DEV)
    lse = torch.empty(B, Hq, dtype=torch.float32, device=DEV)
    ws = torch.empty(hydra.attn_workspace_bytes(t["q"], P, S, Hkv), dtype=torch.uint8, device=DEV)
    side = torch.cuda.Stream() if aux else None

    def step():
        hydra.append_kv(k_in, v_in, t["sk"], t["sv"], t["lens"])
        H.hydragen_attention(t["q"], t["pk"], t["pv"], t["sk"], t["sv"], t["lens"], out=out, lse_out=lse,
                                 workspace=ws, aux_stream=side)

    # capture on a scratch copy of the state, then restore: capture runs the step once
    state = [x.clone() for x in (t["sk"], t["sv"], t["lens"])]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        k_in.copy_(new_k[0]); v_in.copy_(new_v[0])
        step()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    for x, x0 in zip((t["sk"], t["sv"], t["lens"]), state):
        x.copy_(x0)
    torch.cuda.synchronize()
    for i in range(steps):
        k_in.copy_(new_k[i]); v_in.copy_(new_v[i])
        out.fill_(float("nan")); lse.fill_(float("nan")); ws.fill_(0xFF)  # unwritten rows fail
        g.replay()
        torch.cuda.synchronize()
        lens = t["lens"].cpu().numpy()
        assert (lens == np.minimum(lens0 + i + 1, S)).all()
        cur = dataclasses.replace(pb, sk=_bits(t["sk"]), sv=_bits(t["sv"]), lens=lens.astype(np.int32))
        ref, lref = oracle.flat_attention(cur)
        assert_parity(out, ref, lse, lref, what=f"decode step {i}")
