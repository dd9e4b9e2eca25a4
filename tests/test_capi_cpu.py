"""C-ABI boundary checks that need no GPU: the library loads, exports every symbol
include/hydra.h declares, and rejects bad host-visible arguments synchronously
(nothing is launched on a non-OK status)."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2402_05099_b200 as hydra
from paper_2402_05099_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2402_05099_b200 import build

    build.build()
    return _lib.load()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "hydra.h")).read()
    return sorted(set(re.findall(r"HYDRA_API[^;(]*?\b(hydra_\w+)\s*\(", src)))


def test_header_declares_the_paper_boundary():
    syms = declared_symbols()
    for s in ("hydra_prefix_attn", "hydra_suffix_attn", "hydra_combine", "hydra_tree_attn", "hydra_attn"):
        assert s in syms
    assert sorted(_lib.EXPORTED) == syms


def test_library_exports_every_declared_symbol(lib):
    for s in declared_symbols():
        assert hasattr(lib, s), s
    out = os.popen(f"nm -D {_lib.LIB_PATH}").read()
    for s in declared_symbols():
        assert re.search(rf"\bT {s}\b", out), f"{s} not exported"


def test_library_contains_sm100a_tensor_core_code(lib):
    sass = os.popen(f"cuobjdump -sass {_lib.LIB_PATH} 2>/dev/null").read()
    if not sass:
        pytest.skip("cuobjdump unavailable")
    assert "UTCHMMA" in sass  # tcgen05.mma
    assert "UTMALDG" in sass  # TMA tensor loads
    assert "LDTM" in sass and "STTM" in sass  # tcgen05.ld / st
    assert "HMMA" not in sass.replace("UTCHMMA", "")  # no legacy mma.sync path


def test_version(lib):
    assert "sm_100a" in hydra.version()


def H(Hq=4, Hkv=2, d=128, dtype=_lib.HYDRA_BF16, scale=0.0):
    return _lib.Heads(Hq, Hkv, d, scale, dtype)


FAKE = 1 << 20  # 16-B aligned non-null pointer value; never dereferenced (validation fails first)


def prefix_call(lib, h, B=2, P=8, q=FAKE, k=FAKE, v=FAKE, qsb=512, qsh=128, kst=256, ksh=128):
    return lib.hydra_prefix_attn(ctypes.byref(h), B, q, qsb, qsh, P, k, v, kst, ksh, FAKE, FAKE, None, 0, None)


def test_validation_errors(lib):
    assert prefix_call(lib, H(Hq=3, Hkv=2)) == _lib.HYDRA_ESHAPE  # Hq % Hkv != 0
    assert "Hq % Hkv" in _lib.load().hydra_last_error().decode()
    assert prefix_call(lib, H(), B=0) == _lib.HYDRA_ESHAPE  # B == 0
    assert prefix_call(lib, H(d=96)) == _lib.HYDRA_EUNSUPPORTED
    assert prefix_call(lib, H(d=256, dtype=_lib.HYDRA_F32)) == _lib.HYDRA_EUNSUPPORTED
    assert prefix_call(lib, H(dtype=7)) == _lib.HYDRA_EUNSUPPORTED
    assert prefix_call(lib, H(), q=None) == _lib.HYDRA_EINVAL
    assert prefix_call(lib, H(), q=FAKE + 2) == _lib.HYDRA_EINVAL  # misaligned base
    assert prefix_call(lib, H(), kst=129) == _lib.HYDRA_EINVAL  # misaligned stride
    assert prefix_call(lib, H(), P=-1) == _lib.HYDRA_ESHAPE
    h = H()
    assert lib.hydra_suffix_attn(ctypes.byref(h), 2, FAKE, 512, 128, FAKE, FAKE, 4096, 256, 128, 16, None, FAKE,
                                 FAKE, None, 0, None) == _lib.HYDRA_EINVAL  # lens missing
    assert lib.hydra_combine(4, 128, 0, FAKE, 1, 512, FAKE, 4, FAKE, 0, None, None) == _lib.HYDRA_ESHAPE
    assert lib.hydra_combine(4, 128, 2, FAKE, 0, 512, FAKE, 4, FAKE, 0, None, None) == _lib.HYDRA_EUNSUPPORTED
    assert lib.hydra_combine(4, 128, 2, FAKE, 1, 100, FAKE, 4, FAKE, 0, None, None) == _lib.HYDRA_ESHAPE
    # workspace too small for the composite
    h = H(Hq=40, Hkv=40)
    need = lib.hydra_workspace_size(_lib.HYDRA_OP_ATTN, ctypes.byref(h), 1024, 16384, 256, 0)
    assert need >= 2 * 1024 * 40 * 129 * 4
    st = lib.hydra_attn(ctypes.byref(h), 1024, FAKE, 40 * 128, 128, 16384, FAKE, FAKE, 40 * 128, 128, FAKE, FAKE,
                        256 * 40 * 128, 40 * 128, 128, 256, FAKE, FAKE, 0, None, FAKE, need // 2, None, None)
    assert st == _lib.HYDRA_ENOMEM


def test_config_keys(lib):
    assert lib.hydra_set_config(b"no_such_key", 1) == _lib.HYDRA_EINVAL
    hydra.set_config("prefix_splits", 3)
    assert hydra.get_config("prefix_splits") == 3
    hydra.set_config("prefix_splits", 0)


def _tree(lib, parent, node_len, leaf, node_off=None):
    parent = np.asarray(parent, np.int32)
    node_len = np.asarray(node_len, np.int64)
    node_off = np.zeros_like(node_len) if node_off is None else np.asarray(node_off, np.int64)
    leaf = np.asarray(leaf, np.int32)
    out = ctypes.c_void_p()
    st = lib.hydra_tree_create(parent.ctypes.data, node_off.ctypes.data, node_len.ctypes.data, len(parent),
                               leaf.ctypes.data, len(leaf), ctypes.byref(out))
    return st, _lib.load().hydra_last_error().decode()


def test_tree_validation(lib):
    """S:215-223 validate(): the violations are reported before anything touches the GPU."""
    assert _tree(lib, [-1, -1], [4, 4], [1])[0] == _lib.HYDRA_ESHAPE  # multiple roots
    assert "multiple roots" in _tree(lib, [-1, -1], [4, 4], [1])[1]
    assert _tree(lib, [1, 2, 1], [4, 4, 4], [0])[0] == _lib.HYDRA_ESHAPE  # no root / cycle
    assert _tree(lib, [-1, 0, 0], [4, 0, 3], [1, 2])[0] == _lib.HYDRA_ESHAPE  # empty non-root node
    assert _tree(lib, [-1, 0, 0], [4, 2, 3], [0, 2])[0] == _lib.HYDRA_ESHAPE  # sequence on a non-leaf
    assert _tree(lib, [-1, 0, 0], [4, 2, 3], [2, 2])[0] == _lib.HYDRA_ESHAPE  # leaf 1 unused
    assert _tree(lib, [-1, 5], [4, 2], [1])[0] == _lib.HYDRA_ESHAPE  # parent out of range
    assert _tree(lib, [-1, 0], [4, 2], [7])[0] == _lib.HYDRA_ESHAPE  # leaf out of range


def test_python_api_refuses_cpu_tensors():
    import torch

    q = torch.zeros(2, 4, 128, dtype=torch.bfloat16)
    k = torch.zeros(8, 2, 128, dtype=torch.bfloat16)
    with pytest.raises(ValueError, match="CUDA"):
        hydra.prefix_attn(q, k, k)


def test_paged_validation_errors(lib):
    """hydra_paging checks (include/hydra.h): page_size a power of two >= 8, n_pages >= 1,
    S_cap <= bt_stride * page_size, non-null table -- all rejected before any launch."""
    h = H()

    def suffix(pg, S_cap=64):
        return lib.hydra_suffix_attn_paged(ctypes.byref(h), 2, FAKE, 512, 128, FAKE, FAKE, 16 * 2 * 128, 2 * 128,
                                           128, ctypes.byref(pg) if pg is not None else None, S_cap, FAKE, FAKE,
                                           FAKE, None, 0, None)

    P = _lib.Paging
    assert suffix(None) == _lib.HYDRA_EINVAL
    assert suffix(P(None, 4, 16, 8)) == _lib.HYDRA_EINVAL  # null block table
    assert suffix(P(FAKE, 4, 12, 8)) == _lib.HYDRA_ESHAPE  # not a power of two
    assert suffix(P(FAKE, 8, 4, 8)) == _lib.HYDRA_ESHAPE  # below 8 tokens
    assert suffix(P(FAKE, 4, 16, 0)) == _lib.HYDRA_ESHAPE  # empty pool
    assert suffix(P(FAKE, 3, 16, 8)) == _lib.HYDRA_ESHAPE  # 3 * 16 < S_cap = 64
    assert "bt_stride" in lib.hydra_last_error().decode()
    assert lib.hydra_append_kv_paged(ctypes.byref(h), 2, FAKE, FAKE, 256, 128, FAKE, FAKE, 4096, 256, 128, None, 64,
                                     FAKE, None) == _lib.HYDRA_EINVAL
    assert lib.hydra_append_kv_paged(ctypes.byref(h), 2, FAKE, FAKE, 256, 128, FAKE, FAKE, 4096, 256, 128,
                                     ctypes.byref(P(FAKE, 2, 16, 8)), 64, FAKE, None) == _lib.HYDRA_ESHAPE
    need = lib.hydra_workspace_size(_lib.HYDRA_OP_ATTN, ctypes.byref(h), 2, 256, 64, 0)
    assert lib.hydra_attn_paged(ctypes.byref(h), 2, FAKE, 512, 128, 256, FAKE, FAKE, 256, 128, FAKE, FAKE, 4096, 256,
                                128, ctypes.byref(P(FAKE, 4, 24, 8)), 64, FAKE, FAKE, 0, None, FAKE, need, None,
                                None) == _lib.HYDRA_ESHAPE


# ---------------------------------------------------------------- release vs testing build
def _kernel_symbols(path):
    out = os.popen(f"cuobjdump -elf {path} 2>/dev/null").read()
    return set(re.findall(r"_ZN5hydra\w+", out))


def test_release_library_has_no_wrong_result_modes(lib):
    """The release libhydra.so carries none of the testing build's wrong-result paths: no
    no-exp instantiation of the persistent prefix kernel (kPolyEvery = -1), and the
    timing-experiment / sabotage / trace switches are rejected (include/hydra.h)."""
    syms = _kernel_symbols(_lib.RELEASE_LIB)
    if not syms:
        pytest.skip("cuobjdump unavailable")
    assert any("prefix_tc2_kernel" in s for s in syms)
    assert not any("prefix_tc2_kernelILin1" in s for s in syms), "no-exp timing variant shipped in release"
    test_syms = _kernel_symbols(_lib.TEST_LIB)
    assert any("prefix_tc2_kernelILin1" in s for s in test_syms)  # the testing build keeps it
    for key in (b"tc_debug_variant", b"prefix_trace", b"suffix_trace", b"inject_combine_bug", b"mutate"):
        assert lib.hydra_set_config(key, 1) == _lib.HYDRA_EINVAL
        assert "testing build" in lib.hydra_last_error().decode()
    assert lib.hydra_set_config(b"prefix_poly", -1) == _lib.HYDRA_OK and hydra.get_config("prefix_poly") == 4
    assert hydra.get_config("testing_build") == 0
    assert lib.hydra_debug_lens_violations(0) == -1  # no device check in release (kernels clamp)
    assert "testing" not in hydra.version()


def test_testing_library_accepts_test_switches():
    """libhydra_test.so in a subprocess (HYDRA_TESTING=1): the sabotage keys exist there."""
    import subprocess
    import sys

    code = ("import paper_2402_05099_b200 as h; from paper_2402_05099_b200 import _lib;"
            "assert _lib.LIB_PATH == _lib.TEST_LIB; assert h.get_config('testing_build') == 1;"
            "h.set_config('inject_combine_bug', 1); h.set_config('mutate', 2); assert h.get_config('mutate') == 2;"
            "assert 'testing' in h.version(); print('ok')")
    env = dict(os.environ, HYDRA_TESTING="1")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr


def test_config_is_thread_local(lib):
    """hydra_set_config is per thread (hydra.h "Thread safety"): another thread's switch does
    not leak into this thread's calls."""
    import threading

    hydra.set_config("prefix_splits", 5)
    seen = {}

    def other():
        seen["before"] = hydra.get_config("prefix_splits")
        hydra.set_config("prefix_splits", 9)
        seen["after"] = hydra.get_config("prefix_splits")

    t = threading.Thread(target=other)
    t.start()
    t.join()
    assert seen == {"before": 0, "after": 9}
    assert hydra.get_config("prefix_splits") == 5
    hydra.set_config("prefix_splits", 0)


def test_workspace_parts_op(lib):
    """HYDRA_OP_PARTS sizes n_parts caller-staged partial slots (the n_parts argument)."""
    h = H(Hq=8, Hkv=2)
    one = 3 * 8 * (128 + 1) * 4
    assert lib.hydra_workspace_size(_lib.HYDRA_OP_PARTS, ctypes.byref(h), 3, 0, 0, 1) == one
    assert lib.hydra_workspace_size(_lib.HYDRA_OP_PARTS, ctypes.byref(h), 3, 0, 0, 5) == 5 * one
    assert lib.hydra_workspace_size(_lib.HYDRA_OP_PARTS, ctypes.byref(h), 3, 0, 0, 0) == 0
