"""Test helpers: move synth problems to the GPU and compare with the oracle."""
from __future__ import annotations

import numpy as np
import torch

# Gates (BASELINE.json north_star)
BF16_MAX, BF16_MEAN, BF16_LSE = 2e-2, 2e-3, 1e-3
F32_TOL = 1e-5


def to_torch(a: np.ndarray, dtype: str, device) -> torch.Tensor:
    if dtype == "bf16":
        return torch.from_numpy(np.ascontiguousarray(a)).view(torch.bfloat16).to(device)
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(device)


def problem_to(pb, device):
    t = {n: to_torch(getattr(pb, n), pb.dtype, device) for n in ("q", "pk", "pv", "sk", "sv")}
    t["lens"] = torch.from_numpy(pb.lens.astype(np.int32)).to(device)
    return t


def tree_to(tp, device):
    t = {n: to_torch(getattr(tp, n), tp.dtype, device) for n in ("q", "node_k", "node_v", "sk", "sv")}
    t["lens"] = torch.from_numpy(tp.lens.astype(np.int32)).to(device)
    return t


def errors(out: torch.Tensor, ref: np.ndarray):
    o = out.float().cpu().numpy().astype(np.float64)
    d = np.abs(o - ref)
    return float(np.nanmax(d)) if d.size else 0.0, float(np.mean(d)) if d.size else 0.0, bool(np.isfinite(o).all())


def lse_err(lse: torch.Tensor, ref: np.ndarray) -> float:
    l = lse.float().cpu().numpy().astype(np.float64)
    fin = np.isfinite(ref)
    assert (np.isneginf(l) == np.isneginf(ref)).all(), "empty-set sentinel mismatch"
    return float(np.max(np.abs(l[fin] - ref[fin]))) if fin.any() else 0.0


def assert_parity(out, ref, lse=None, lse_ref=None, dtype="bf16", what=""):
    mx, mean, finite = errors(out, ref)
    assert finite, f"{what}: non-finite output"
    if dtype == "bf16":
        assert mx <= BF16_MAX and mean <= BF16_MEAN, f"{what}: max {mx:.3e} mean {mean:.3e}"
        if lse is not None:
            le = lse_err(lse, lse_ref)
            assert le <= BF16_LSE, f"{what}: lse err {le:.3e}"
    else:
        assert mx <= F32_TOL, f"{what}: max {mx:.3e}"
        if lse is not None:
            le = lse_err(lse, lse_ref)
            assert le <= F32_TOL, f"{what}: lse err {le:.3e}"
    return mx, mean
