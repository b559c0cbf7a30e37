"""The C-ABI boundary without a GPU: the library loads, exports every symbol
include/tt.h declares, and rejects bad arguments on the host before any CUDA
call (so none of these tests touches a device)."""
import ctypes
import math
import os
import re

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DT = [torch.float32, torch.float16, torch.bfloat16]
FAKE = 0x10000  # 16-B aligned, never dereferenced: validation fails first


def _declared():
    names = set()
    for h in os.listdir(os.path.join(ROOT, "include")):
        if h.endswith(".h"):
            src = open(os.path.join(ROOT, "include", h)).read()
            names |= set(re.findall(r"TT_API\s+[\w\s\*]+?\b(ttx?_\w+)\s*\(", src))
    return names


def test_header_declares_expected_api(ttlib):
    decl = _declared()
    assert decl == set(ttlib.EXPORTS), decl ^ set(ttlib.EXPORTS)


def test_library_exports_every_declared_symbol(ttlib):
    L = ttlib.lib()
    for name in _declared():
        assert hasattr(L, name), name
        assert ctypes.cast(getattr(L, name), ctypes.c_void_p).value


def test_library_is_sm100a_only():
    from paper_2010_05680_b200 import build as b
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", b.LIB],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    ptx = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-ptx", b.LIB],
                         capture_output=True, text=True).stdout
    assert "compute_100." not in ptx.replace("compute_100a", "")


def test_status_strings_and_version(ttlib):
    assert ttlib.status_string(0) == "TT_SUCCESS"
    assert ttlib.status_string(1) == "TT_ERROR_INVALID_VALUE"
    assert ttlib.status_string(2) == "TT_ERROR_NOT_SUPPORTED"
    assert ttlib.status_string(3) == "TT_ERROR_CUDA"
    assert ttlib.version() >= 10000
    assert ttlib.lib().tt_last_cuda_error() == 0


@pytest.mark.parametrize("dtype", DT)
def test_softmax_validation(ttlib, dtype):
    f = ttlib.tt_softmax_masked_raw
    INV, NS, OK = 1, 2, 0
    assert f(dtype, 0, 0, 2, 2, 2, 8, 1.0) == INV                 # null pointers
    assert f(dtype, FAKE, 0, 2, 2, 2, 8, 1.0) == INV              # null lengths
    assert f(dtype, FAKE, FAKE, -1, 2, 2, 8, 1.0) == INV          # negative dim
    assert f(dtype, FAKE, FAKE, 2, 2, 2, -8, 1.0) == INV
    assert f(dtype, FAKE, FAKE, 2, 2, 2, 8, math.inf) == INV      # non-finite scale
    assert f(dtype, FAKE, FAKE, 2, 2, 2, 8, math.nan) == INV
    assert f(dtype, FAKE, FAKE, 1 << 40, 1 << 20, 1 << 10, 8, 1.0) == INV   # overflow
    assert f(dtype, FAKE + 2, FAKE, 2, 2, 2, 8, 1.0) == NS        # misaligned base
    assert f(dtype, FAKE, FAKE + 1, 2, 2, 2, 8, 1.0) == NS        # misaligned lengths
    assert f(dtype, FAKE, FAKE, 2, 2, 2, ttlib.TT_MAX_SOFTMAX_COLS + 1, 1.0) == NS
    # empty problems: success, no CUDA call, null pointers allowed
    for shape in ((0, 2, 2, 8), (2, 0, 2, 8), (2, 2, 0, 8), (2, 2, 2, 0)):
        assert f(dtype, 0, 0, *shape, 1.0) == OK


@pytest.mark.parametrize("dtype", DT)
def test_layernorm_validation(ttlib, dtype):
    f = ttlib.tt_add_bias_layernorm_raw
    INV, NS, OK = 1, 2, 0
    e = 4 if dtype == torch.float32 else 2
    rows, hid = 4, 64
    n = rows * hid * e
    out, x, r = FAKE, FAKE + 4 * n, FAKE + 8 * n
    b, g, be = FAKE + 12 * n, FAKE + 12 * n + 4096, FAKE + 12 * n + 8192
    ok = (out, x, r, b, g, be)
    assert f(dtype, 0, x, r, b, g, be, rows, hid, 1e-5) == INV
    assert f(dtype, out, x, r, b, 0, be, rows, hid, 1e-5) == INV
    assert f(dtype, *ok, -1, hid, 1e-5) == INV
    assert f(dtype, *ok, rows, hid, -1e-5) == INV                 # negative eps
    assert f(dtype, *ok, rows, hid, math.inf) == INV
    assert f(dtype, *ok, rows, hid, math.nan) == INV
    assert f(dtype, *ok, 1 << 62, 1 << 10, 1e-5) == INV           # overflow
    # out partially overlapping x (exact aliasing is allowed, tested on GPU)
    assert f(dtype, x + 64, x, r, b, g, be, rows, hid, 1e-5) == INV
    assert f(dtype, r - 64, x, r, b, g, be, rows, hid, 1e-5) == INV
    # parameters overlapping the output
    assert f(dtype, out, x, r, out + 16, g, be, rows, hid, 1e-5) == INV
    assert f(dtype, out + 2, x, r, b, g, be, rows, hid, 1e-5) == NS
    assert f(dtype, out, x, r, b, g, be + 8, rows, hid, 1e-5) == NS
    big = 1 << 24  # far-apart fake buffers for the oversized-row check
    far = tuple(FAKE + i * big for i in range(6))
    assert f(dtype, *far, rows, ttlib.TT_MAX_LN_HIDDEN + 1, 1e-5) == NS
    assert f(dtype, 0, 0, 0, 0, 0, 0, 0, hid, 1e-5) == OK
    assert f(dtype, 0, 0, 0, 0, 0, 0, rows, 0, 1e-5) == OK


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-device error path")
def test_launch_without_device_fails_loudly(ttlib):
    """With valid arguments and no GPU the call reaches the launch and returns
    TT_ERROR_CUDA: there is no CPU fallback."""
    st = ttlib.tt_softmax_masked_raw(torch.float32, FAKE, FAKE, 1, 1, 1, 8, 1.0)
    assert st == ttlib.TT_ERROR_CUDA
    assert ttlib.lib().tt_last_cuda_error() != 0
    with pytest.raises(RuntimeError):
        import paper_2010_05680_b200._lib as L
        L._check(st, "x")


@pytest.mark.parametrize("dtype,Sk,tier", [
    (torch.float32, 40, "softmax_warp<f32,V16,G16,NV1,T256,M6,P4>"),
    (torch.float16, 37, "softmax_warp<f16,V16,G8,NV1,T256,M6,P4>"),
    (torch.bfloat16, 512, "softmax_warp<bf16,V32,G32,NV1,T256,M6,P4>"),
    (torch.float16, 491, "softmax_warp<f16,V32,G32,NV1,T256,M6,P2>"),
    (torch.float32, 500, "softmax_warp<f32,V32,G32,NV2,T256,M3,P2>"),
    (torch.float32, 4096, "softmax_rows<f32,V32,G128,NV4,R1,T128,M1>"),
    (torch.bfloat16, 16384, "softmax_rows<bf16,V32,G512,NV2,R1,T512,M1>"),
    (torch.bfloat16, 16385, "softmax_cluster<bf16,V32,NV2,T512,C8>"),
    (torch.float32, 131072, "softmax_cluster<f32,V32,NV4,T512,C8>"),
    (torch.float32, 131073, "softmax_long<f32,V16,T256,M4,K65536>"),
    (torch.bfloat16, 1 << 24, "softmax_long<bf16,V16,T256,M4,K65536>"),
])
def test_softmax_tier_plan(ttlib, dtype, Sk, tier):
    assert ttlib.softmax_plan(dtype, 2, 12, 3, Sk) == tier


@pytest.mark.parametrize("dtype,rows,hidden,tier", [
    (torch.float32, 10, 768, "ln_rows<f32,V32,G128,NV4,R1,T128,M1>"),
    (torch.float32, 2000, 768, "ln_rows<f32,V32,G32,NV3,R1,T256,M1,E>"),
    (torch.float32, 30000, 768, "ln_rows<f32,V32,G32,NV3,R1,T128,M1>"),
    (torch.float32, 10000, 768, "ln_rows<f32,V32,G32,NV3,R1,T128,M1>"),
    (torch.float16, 10000, 768, "ln_rows<f16,V16,G32,NV3,R1,T128,M1>"),
    (torch.float16, 10, 768, "ln_rows<f16,V32,G128,NV2,R1,T128,M1>"),
    (torch.float16, 800, 768, "ln_rows<f16,V16,G128,NV4,R1,T128,M1>"),
    (torch.float16, 2000, 768, "ln_rows<f16,V32,G32,NV2,R1,T128,M1,E>"),
    (torch.float16, 30000, 768, "ln_warp<f16,V16,G32,NV3,T256,M3,PF0>"),
    (torch.float16, 6000, 768, "ln_rows<f16,V32,G16,NV3,R1,T256,M1>"),   # one-wave band
    (torch.bfloat16, 7000, 768, "ln_rows<bf16,V32,G16,NV3,R1,T256,M1>"),
    (torch.float16, 11000, 768, "ln_rows<f16,V16,G32,NV3,R1,T128,M1>"),
    (torch.float16, 12000, 768, "ln_warp<f16,V16,G32,NV3,T256,M3,PF0>"),  # kSmallRows = 11500
    (torch.bfloat16, 31808, 768, "ln_warp<bf16,V16,G32,NV3,T256,M3,PF0>"),
    (torch.bfloat16, 10, 1024, "ln_rows<bf16,V32,G32,NV2,R1,T256,M1,E>"),
    (torch.bfloat16, 32768, 1024, "ln_rows<bf16,V32,G32,NV2,R1,T64,M12>"),
    (torch.float32, 10, 37, "ln_rows<f32,V4,G32,NV4,R1,T256,M1>"),
    (torch.float16, 10, 16, "ln_warp<f16,V16,G4,NV1,T256,M4,PF0>"),
    (torch.float32, 10, 4096, "ln_rows<f32,V32,G128,NV4,R1,T128,M1>"),
])
def test_layernorm_tier_plan(ttlib, dtype, rows, hidden, tier):
    assert ttlib.layernorm_plan(dtype, rows, hidden) == tier


def test_tier_enumeration_and_force(ttlib):
    for op in ("softmax", "layernorm"):
        for dt in DT:
            names = ttlib.tiers(op, dt)
            assert len(names) >= 10 and all(names)
    with pytest.raises(ttlib.TTError):
        ttlib.force_tier("softmax", torch.float32, 10 ** 6)
    ttlib.force_tier("softmax", torch.bfloat16, 0)   # G4 tier cannot serve Sk=512
    try:
        assert ttlib.softmax_plan(torch.bfloat16, 1, 1, 1, 512) == \
            "softmax_warp<bf16,V32,G32,NV1,T256,M6,P4>"
        assert ttlib.softmax_plan(torch.bfloat16, 1, 1, 1, 8) == ttlib.tiers("softmax", torch.bfloat16)[0]
    finally:
        ttlib.force_tier("softmax", torch.bfloat16, -1)


@pytest.mark.parametrize("dtype", DT)
def test_packed_validation(ttlib, dtype):
    L = ttlib.lib()
    f = getattr(L, f"tt_softmax_packed_{ {torch.float32: 'f32', torch.float16: 'f16', torch.bfloat16: 'bf16'}[dtype]}")
    INV, NS, OK = 1, 2, 0
    cap = 1024 if dtype == torch.float32 else 2048
    assert f(0, FAKE, FAKE, 4, 12, 100, 50, 1.0, 0) == INV              # null scores
    assert f(FAKE, 0, FAKE, 4, 12, 100, 50, 1.0, 0) == INV
    assert f(FAKE, FAKE, 0, 4, 12, 100, 50, 1.0, 0) == INV
    assert f(FAKE, FAKE, FAKE, -1, 12, 100, 50, 1.0, 0) == INV
    assert f(FAKE, FAKE, FAKE, 4, 12, 100, 50, float("nan"), 0) == INV
    assert f(FAKE + 2, FAKE, FAKE, 4, 12, 100, 50, 1.0, 0) == NS
    assert f(FAKE, FAKE + 2, FAKE, 4, 12, 100, 50, 1.0, 0) == NS
    assert f(FAKE, FAKE, FAKE + 4, 4, 12, 100, 50, 1.0, 0) == NS
    assert f(FAKE, FAKE, FAKE, 4, 12, 100, cap + 1, 1.0, 0) == NS
    assert f(FAKE, FAKE, FAKE, 4, 1 << 20, 1 << 13, 50, 1.0, 0) == NS   # rows >= 2^32
    for args in ((0, 12, 100, 50), (4, 0, 100, 50), (4, 12, 0, 50), (4, 12, 100, 0)):
        assert f(0, 0, 0, *args, 1.0, 0) == OK
    assert ttlib.softmax_packed_plan(dtype, 512).startswith("softmax_packed<")


def test_staged_overlap_validation(ttlib):
    """Host-side validation of the overlapped staging calls (include/tt.h): bad
    arguments are rejected before any CUDA call; empty problems are no-ops."""
    L = ttlib.lib()
    INV, OK = 1, 0
    fs = L.tt_softmax_masked_staged_overlap
    # null host buffers, with a distinct copy stream and several chunks
    assert fs(1, 0, 0, FAKE, FAKE, 2, 2, 2, 8, 1.0, 4, 0, FAKE) == INV
    assert fs(1, FAKE, FAKE, 0, FAKE, 2, 2, 2, 8, 1.0, 4, 0, FAKE) == INV       # null device
    assert fs(1, FAKE, FAKE, FAKE, FAKE, 2, 2, 2, 8, math.nan, 4, 0, FAKE) == INV
    assert fs(1, 0, 0, 0, 0, 0, 2, 2, 8, 1.0, 4, 0, FAKE) == OK                 # empty
    fl = L.tt_add_bias_layernorm_staged_overlap
    assert fl(2, 0, 0, 0, FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, 4, 64, 1e-5, 4, 0, FAKE) == INV
    assert fl(2, FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, 4, 64, -1.0, 4, 0,
              FAKE) == INV                                                      # eps < 0
    assert fl(2, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 64, 1e-5, 4, 0, FAKE) == OK      # empty
    # dev_x and dev_residual are both H2D targets: overlap is rejected
    F2 = FAKE + (1 << 24)
    for f, extra in ((fl, (4, 0, FAKE)), (L.tt_add_bias_layernorm_staged, (0,))):
        args = (2, FAKE, FAKE, FAKE, F2, FAKE, FAKE + 64, F2 + (1 << 20), F2 + (1 << 21),
                F2 + (1 << 22), 4, 64, 1e-5)
        assert f(*args, *extra) == INV


def test_softmax_preference_row_threshold(ttlib):
    """Small fp32 rows pick the 8-lane multi-vector tiers only for calls of more
    than 2048 rows (C2), not for C1-sized calls (DESIGN §5 "Small fp32 rows")."""
    f32 = torch.float32
    assert ttlib.softmax_plan(f32, 20, 12, 40, 40) == "softmax_warp<f32,V16,G8,NV2,T256,M6,P4>"
    assert ttlib.softmax_plan(f32, 1, 12, 40, 40) == "softmax_warp<f32,V16,G16,NV1,T256,M6,P4>"
    assert ttlib.softmax_plan(f32, 20, 12, 100, 100) == "softmax_warp<f32,V16,G8,NV4,T256,M3,P4,F>"
    # LayerNorm bands at hidden 768: one CTA per row up to 1024 rows
    assert ttlib.layernorm_plan(f32, 40, 768) == "ln_rows<f32,V32,G128,NV4,R1,T128,M1>"
    assert ttlib.layernorm_plan(f32, 5000, 768) == "ln_rows<f32,V32,G32,NV3,R1,T128,M1>"


def test_every_preferred_tier_is_compiled(ttlib):
    """Every tier the preference tables name (softmax.cu kSmPref, layernorm.cu
    kLnPref*) exists in the product library -- a name missing from it would
    silently fall back to the generic rule."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    csrc = os.path.join(root, "paper_2010_05680_b200", "csrc")
    dn = {"f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16}
    for op, fname in (("softmax", "softmax.cu"), ("layernorm", "layernorm.cu")):
        names = re.findall(r'"((?:softmax|ln)_\w+<(f32|f16|bf16),[^"]*>)"', open(os.path.join(csrc, fname)).read())
        names = [(n, d) for n, d in names if "," in n and "TN" not in n]
        assert names, fname
        for n, d in names:
            assert n in ttlib.tiers(op, dn[d]), n
    for op in ("softmax", "layernorm"):
        for dt in dn.values():
            names = ttlib.tiers(op, dt)
            assert len(names) == len(set(names)), (op, dt)   # one entry per kernel
