"""Host-side validation of the NEXT-2 entry points (no GPU needed: every case
returns before any CUDA call)."""
import pytest

FAKE = 0x10000
INV, NS, OK = 1, 2, 0


@pytest.mark.parametrize("dt", [0, 1, 2])
def test_gelu_validation(ttlib, dt):
    f = ttlib.lib().tt_add_bias_gelu
    e = 4 if dt == 0 else 2
    far = 1 << 24
    assert f(dt, 0, FAKE, FAKE + far, 4, 8, 0, 0) == INV
    assert f(dt, FAKE, FAKE + far, FAKE + 2 * far, -1, 8, 0, 0) == INV
    assert f(dt, FAKE, FAKE + far, FAKE + 2 * far, 4, 8, 2, 0) == INV      # approximate flag
    assert f(3, FAKE, FAKE + far, FAKE + 2 * far, 4, 8, 0, 0) == INV       # dtype
    assert f(dt, FAKE + e, FAKE, FAKE + far, 4, 8, 0, 0) == INV            # partial alias
    assert f(dt, FAKE, FAKE + far, FAKE + 4, 4, 8, 0, 0) == INV            # bias inside out
    assert f(dt, FAKE + 1, FAKE + 1 + far, FAKE + 2 * far, 4, 8, 0, 0) == NS
    assert f(dt, 0, 0, 0, 0, 8, 0, 0) == OK and f(dt, 0, 0, 0, 4, 0, 1, 0) == OK


@pytest.mark.parametrize("dt", [0, 1, 2])
def test_split_merge_validation(ttlib, dt):
    s = ttlib.lib().tt_split_qkv_add_bias
    m = ttlib.lib().tt_merge_heads
    far = 1 << 24
    P = [FAKE + i * far for i in range(5)]
    assert s(dt, 0, P[1], P[2], P[3], P[4], 1, 2, 3, 8, 0) == INV
    assert s(dt, P[0], P[0], P[2], P[3], P[4], 1, 2, 3, 8, 0) == INV       # q == k
    assert s(dt, P[0], P[1], P[3], P[3], P[4], 1, 2, 3, 8, 0) == INV       # v over qkv
    assert s(dt, *P, -1, 2, 3, 8, 0) == INV
    assert s(dt, P[0] + 1, P[1], P[2], P[3], P[4], 1, 2, 3, 8, 0) == NS
    huge = [FAKE + i * (1 << 42) for i in range(5)]                        # no overlap
    assert s(dt, *huge, 1 << 12, 1 << 12, 64, 64, 0) == NS                 # > 2^32 items
    assert s(dt, 0, 0, 0, 0, 0, 0, 2, 3, 8, 0) == OK
    assert m(dt, 0, P[1], 1, 2, 3, 8, 0) == INV
    assert m(dt, P[0], P[0] + 8, 1, 2, 3, 8, 0) == INV                     # overlap
    assert m(dt, P[0] + 1, P[1], 1, 2, 3, 8, 0) == NS
    assert m(dt, 0, 0, 1, 0, 3, 8, 0) == OK


@pytest.mark.parametrize("dt", [1, 2])
def test_attention_validation(ttlib, dt):
    """tt_attention_fwd (NEXT-3) host checks: every case returns before a CUDA call."""
    f = ttlib.lib().tt_attention_fwd
    far = 1 << 24
    o, q, k, v, L = (FAKE + i * far for i in range(5))
    assert f(dt, o, q, k, v, L, 2, 2, 8, 64, float("nan"), 0) == INV       # scale
    assert f(dt, o, q, k, v, L, -1, 2, 8, 64, 0.125, 0) == INV             # negative dim
    assert f(3, o, q, k, v, L, 2, 2, 8, 64, 0.125, 0) == INV               # dtype
    assert f(dt, 0, q, k, v, L, 2, 2, 8, 64, 0.125, 0) == INV              # null out
    assert f(dt, o, q, k, v, 0, 2, 2, 8, 64, 0.125, 0) == INV              # null lengths
    assert f(dt, o, o + 64, k, v, L, 2, 2, 8, 64, 0.125, 0) == INV         # out overlaps q
    assert f(dt, o, q, k, v, L, 2, 2, 8, 32, 0.125, 0) == NS               # head dim 32
    assert f(0, o, q, k, v, L, 2, 2, 8, 64, 0.125, 0) == NS                # fp32
    assert f(dt, o + 2, q, k, v, L, 2, 2, 8, 64, 0.125, 0) == NS           # misaligned out
    assert f(dt, o, q, k, v, L + 2, 2, 2, 8, 64, 0.125, 0) == NS           # misaligned lengths
    assert f(dt, 0, 0, 0, 0, 0, 0, 2, 8, 64, 0.125, 0) == OK               # empty: no-op


def test_attention_variant_hook(ttlib):
    L = ttlib.lib()
    h, ok = L.ttx_attention_variant, L.ttx_attention_variant_ok
    n = L.ttx_attention_variant_count()
    # the product library holds the automatic choice only; the tuning build
    # (ttx_tuning_build) adds variants 1..11
    want = set(range(12)) if ttlib.tuning_build() else {0}
    assert n == 12 and {v for v in range(n) if ok(v)} == want
    for v in range(n):
        assert h(v) == (OK if v in want else INV)
    assert h(-1) == INV and h(n) == INV
    assert h(0) == OK
