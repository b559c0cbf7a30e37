"""GPU parity: tt_softmax_masked_* (CUDA, through the C ABI) vs the fp64 oracle.

Every config is compared element by element on every row: small ones
directly, the larger ones (C2 S > 128, C3, C4, C5 batches, in the launch
configuration bench.py times) by the threaded oracle request by request
(`_parity.softmax_all_rows`); `_sampled_check` (seeded row samples plus
all-row properties: masked bits exactly 0, valid rows sum to 1, no NaN) is
kept for ad-hoc use."""
import numpy as np
import pytest
import torch

import oracle
import workloads as W
import workloads as W_
from _parity import assert_close, masked_bits_zero, softmax_all_rows

pytestmark = pytest.mark.gpu
DT = [torch.float32, torch.float16, torch.bfloat16]
SUM_TOL = {torch.float32: 1e-4, torch.float16: 5e-3, torch.bfloat16: 2e-2}


def _run(tt, x_cpu, lens, scale):
    x = x_cpu.cuda()
    L = torch.as_tensor(np.asarray(lens, dtype=np.int32)).cuda()
    tt.tt_softmax_masked(x, L, scale)
    torch.cuda.synchronize()
    return x


def _full_check(tt, x_cpu, lens, scale, what=""):
    y = _run(tt, x_cpu, lens, scale)
    ref = oracle.softmax_masked(x_cpu, lens, scale)
    assert_close("softmax", x_cpu.dtype, y, ref, what)
    assert masked_bits_zero(y, lens), what
    return y


def _sampled_check(tt, x_dev, lens, scale, nsample=2048, seed=0, what=""):
    """In-place call on a device tensor; oracle on a seeded sample of rows."""
    B, H, Sq, Sk = x_dev.shape
    nrows = B * H * Sq
    g = torch.Generator().manual_seed(seed)
    idx = torch.randint(0, nrows, (min(nsample, nrows),), generator=g)
    idx[0], idx[-1] = 0, nrows - 1
    rows_before = x_dev.view(nrows, Sk)[idx.cuda()].cpu()
    L = torch.as_tensor(np.asarray(lens, dtype=np.int32)).cuda()
    tt.tt_softmax_masked(x_dev, L, scale)
    torch.cuda.synchronize()
    got = x_dev.view(nrows, Sk)[idx.cuda()].cpu()
    row_lens = np.asarray(lens, dtype=np.int32)[(idx // (H * Sq)).numpy()]
    ref = oracle.softmax_rows(rows_before, row_lens, scale)
    assert_close("softmax", x_dev.dtype, got, ref, what)
    # every row: masked bits, sums, finiteness
    assert masked_bits_zero(x_dev, lens), what
    s = x_dev.float().sum(-1)
    lens_t = torch.as_tensor(np.asarray(lens), device=x_dev.device).clamp(0, Sk)
    valid = (lens_t > 0)[:, None, None].expand(B, H, Sq)
    assert torch.isfinite(s).all()
    assert ((s[valid] - 1).abs() <= SUM_TOL[x_dev.dtype]).all(), what
    assert (s[~valid] == 0).all()


# ----------------------------------------------------------------- C1, C2
def test_c1_bert_base_b1_s40(ttlib):
    x = W.scores(1, 12, 40, 40, torch.float32, seed=W.SEED + 1)
    _full_check(ttlib, x, [40], W.SCALE_BERT, "C1")


@pytest.mark.parametrize("dtype", [torch.float16, torch.float32])
@pytest.mark.parametrize("S", W.C2.extra["seqs"])
@pytest.mark.parametrize("ragged", [False, True])
def test_c2_seq_sweep(ttlib, dtype, S, ragged):
    lens = W.lengths_ragged(20, S) if ragged else W.lengths_full(20, S)
    if S <= 128:
        x = W.scores(20, 12, S, S, dtype, seed=W.SEED + 2 + S)
        _full_check(ttlib, x, lens, W.SCALE_BERT, f"C2 S={S}")
    else:
        x = W.scores(20, 12, S, S, dtype, device="cuda", seed=W.SEED + 2 + S)
        _all_rows_check(ttlib, x, lens, W.SCALE_BERT, f"C2 S={S}")


# ----------------------------------------------------------------- C3, C4, C5
def _all_rows_check(tt, x_dev, lens, scale, what):
    """In-place call on a full-size device tensor; every row vs the oracle."""
    before = x_dev.cpu()
    L = torch.as_tensor(np.asarray(lens, dtype=np.int32)).cuda()
    tt.tt_softmax_masked(x_dev, L, scale)
    torch.cuda.synchronize()
    plan = tt.softmax_plan(x_dev.dtype, *x_dev.shape)
    err = softmax_all_rows(before, x_dev, lens, scale, f"{what} [{plan}]")
    print(f"{what}: {plan}: every row, max abs err {err:.3e}")


@pytest.mark.parametrize("dtype", [torch.float16, torch.float32])
def test_c3_variable_length_batch(ttlib, dtype):
    lens = W.c3_lengths()
    S = int(lens.max())
    x = W.scores(64, 12, S, S, dtype, device="cuda", seed=W.SEED + 3)
    _all_rows_check(ttlib, x, lens, W.SCALE_BERT, "C3")


@pytest.mark.parametrize("ragged", [False, True])
def test_c4_bert_large_full_size(ttlib, ragged):
    lens = W.lengths_ragged(64, 512, seed_offset=4) if ragged else W.lengths_full(64, 512)
    x = W.scores(64, 16, 512, 512, torch.bfloat16, device="cuda", seed=W.SEED + 4)
    _all_rows_check(ttlib, x, lens, W.SCALE_BERT, "C4")


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
def test_c5_stream_batches(ttlib, dtype):
    batches = W.c5_stream()
    for bi in (0, 17, 63):
        lens = batches[bi]
        S = int(lens.max())
        x = W.scores(64, 12, S, S, dtype, device="cuda", seed=W.SEED + 5 + bi)
        _all_rows_check(ttlib, x, lens, W.SCALE_BERT, f"C5 b{bi}")


@pytest.mark.parametrize("Sk", [37, 65, 127, 100])
def test_fp32_ragged_many_rows_sub_warp_tiers(ttlib, Sk):
    """fp32 rows of 33..128 keys in calls of more than 2048 rows take the G8
    NV2 / NV4+prefetch tiers (softmax.cu kSmPref); 256 rows per request so
    whole CTAs belong to one request (one-request narrow paths), odd pitches
    (Sk % 4 != 0: head / tail code), poison in the padding."""
    lens = [Sk, 1, 7, 8, 9, 15, 16, 17, 31, 32, 33, Sk // 2, Sk - 1, 0, Sk, 3]
    x = W.scores(len(lens), 4, 64, Sk, torch.float32, seed=Sk + 11)
    plan = ttlib.softmax_plan(torch.float32, len(lens), 4, 64, Sk)
    assert len(lens) * 4 * 64 > 2048
    _full_check(ttlib, x, lens, W.SCALE_BERT, f"fp32 many rows Sk={Sk} [{plan}]")
    xp = W.poison_masked(x, lens)
    _full_check(ttlib, xp, lens, -0.25, f"fp32 many rows poison Sk={Sk} [{plan}]")


# ----------------------------------------------------------------- edge cases
@pytest.mark.parametrize("dtype", DT)
def test_every_row_length_1_to_160(ttlib, dtype):
    """Every Sk 1..160: all tiers' head / body / tail splits and group sizes."""
    for Sk in range(1, 161):
        B = 3
        lens = [Sk, max(Sk // 2, 1), 0]
        # 6 rows per request (requests far smaller than a CTA: per-row lengths)
        # and 64 rows per request (the warp tiers' one-request CTAs)
        for H, Sq in ((2, 3), (4, 16)):
            x = W.scores(B, H, Sq, Sk, dtype, seed=Sk)
            _full_check(ttlib, x, lens, W.SCALE_BERT, f"Sk={Sk} H={H} Sq={Sq}")


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("Sk", [255, 256, 257, 511, 513, 767, 1000, 1023, 1024, 1025, 2047, 2048,
                                2049, 4095, 4096, 4099, 8192, 16384, 16385, 32768, 32771,
                                65536, 100003, 131072, 131073, 262147, 400000])
def test_long_rows_and_tier_boundaries(ttlib, dtype, Sk):
    lens = [Sk, Sk - 1, 1, Sk // 3]
    x = W.scores(4, 1, 2, Sk, dtype, seed=Sk + 7)
    _full_check(ttlib, x, lens, W.SCALE_BERT, f"Sk={Sk}")


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("Sk", [131073, 8 * 65536 + 3, 9 * 65536 + 5])
def test_long_tier_segments_and_masks(ttlib, dtype, Sk):
    """Rows beyond the cluster tier (softmax_long: <= 8 CTAs per row, each making an
    online (m, s) pass and a normalising pass over its key segment, pairs merged
    through distributed shared memory): valid lengths ending inside a segment,
    on segment boundaries, in the first segment only, 0 and 1; odd pitches so
    rows and segments start unaligned; poison in the padding; negative scale."""
    C = min(8, -(-Sk // 65536))  # CTAs per row (softmax.cu launch_softmax_long, K65536)
    Wseg = (-(-Sk // C) + 63) // 64 * 64
    lens = [Sk, 1, 0, Wseg, Wseg + 1, (C - 1) * Wseg - 2, (C - 1) * Wseg, Sk - 1, 17]
    x = W.scores(len(lens), 1, 1, Sk, dtype, seed=Sk)
    assert ttlib.softmax_plan(dtype, len(lens), 1, 1, Sk).startswith("softmax_long<")
    _full_check(ttlib, x, lens, W.SCALE_BERT, "long")
    _full_check(ttlib, W.poison_masked(x, lens), lens, -0.25, "long poison")


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("Sk", [491, 500, 512, 257])
def test_short_requests_narrow_groups(ttlib, dtype, Sk):
    """Requests whose rows fill whole CTAs take the narrow-group path (4/8/16
    lanes per row + zero-filled padding vectors); every boundary of those
    widths, aligned and odd pitches."""
    lens = [1, 5, 31, 32, 33, 63, 64, 65, 127, 128, 129, 200, 255, 256, Sk - 1, Sk, 0]
    x = W.scores(len(lens), 4, 16, Sk, dtype, seed=Sk)
    _full_check(ttlib, x, lens, W.SCALE_BERT, f"narrow Sk={Sk}")
    xp = W.poison_masked(x, lens)
    _full_check(ttlib, xp, lens, -0.25, f"narrow poison Sk={Sk}")


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("Sk", [100, 200, 250, 256, 300, 500])
def test_short_requests_fewer_vectors(ttlib, dtype, Sk):
    """Multi-vector tiers (NV > 1): a CTA whose rows all belong to one short
    request runs them with the fewest vectors per lane that hold L_b keys
    (softmax_narrow_nv).  256 rows per request so that whole CTAs belong to one
    request; lengths at every K * G * VE boundary of the G8 (16-bit) and G32
    (fp32) tiers, aligned and unaligned pitches, poison in the padding."""
    lens = [1, 7, 8, 9, 31, 32, 33, 63, 64, 65, 127, 128, 129, 191, 192, 193, 255, 256, 257,
            Sk - 1, Sk, 0]
    lens = [min(l, Sk) for l in lens]
    x = W.scores(len(lens), 4, 64, Sk, dtype, seed=Sk + 1)
    _full_check(ttlib, x, lens, W.SCALE_BERT, f"fewer-vectors Sk={Sk}")
    xp = W.poison_masked(x, lens)
    _full_check(ttlib, xp, lens, -0.25, f"fewer-vectors poison Sk={Sk}")


@pytest.mark.parametrize("dtype", DT)
def test_length_edge_values(ttlib, dtype):
    Sk = 70
    lens = [0, -5, 1, 69, 70, 71, 1 << 30, -(1 << 30)]
    x = W.scores(len(lens), 2, 2, Sk, dtype, seed=3)
    y = _full_check(ttlib, x, lens, W.SCALE_BERT, "edge lengths")
    assert (y[0] == 0).all() and (y[1] == 0).all() and (y[7] == 0).all()
    assert (y[2, :, :, 0] == 1).all()


@pytest.mark.parametrize("dtype", DT)
def test_poison_in_masked_columns_is_never_read(ttlib, dtype):
    for Sk in (37, 64, 500, 512, 3000):
        lens = [Sk // 2, 1, Sk, 0]
        x = W.scores(4, 2, 3, Sk, dtype, seed=Sk)
        clean = _run(ttlib, x, lens, W.SCALE_BERT)
        dirty = _run(ttlib, W.poison_masked(x, lens), lens, W.SCALE_BERT)
        ib = torch.int32 if dtype == torch.float32 else torch.int16
        assert torch.equal(clean.view(ib), dirty.view(ib)), Sk


@pytest.mark.parametrize("dtype", DT)
def test_peaky_and_scale_variants(ttlib, dtype):
    Sk = 130
    lens = [130, 77]
    x = W.scores(2, 3, 5, Sk, dtype, seed=99, std=40.0)
    for scale in (W.SCALE_BERT, 1.0, -0.5, 0.0, 1e-3):
        _full_check(ttlib, x, lens, scale, f"scale={scale}")


@pytest.mark.parametrize("dtype", DT)
def test_deterministic_bitwise(ttlib, dtype):
    lens = W.c3_lengths(salt=1)
    S = int(lens.max())
    x = W.scores(64, 12, S, S, dtype, device="cuda", seed=5)
    a, b = x.clone(), x.clone()
    L = torch.as_tensor(lens).cuda()
    ttlib.tt_softmax_masked(a, L, W.SCALE_BERT)
    ttlib.tt_softmax_masked(b, L, W.SCALE_BERT)
    torch.cuda.synchronize()
    ib = torch.int32 if dtype == torch.float32 else torch.int16
    assert torch.equal(a.view(ib), b.view(ib))


def test_nondefault_stream_and_offset_views(ttlib):
    """A side stream, and a base pointer 16 B (not 32 B) aligned."""
    s = torch.cuda.Stream()
    Sk = 512
    buf = W.scores(1, 1, 1, 8 + 2 * 3 * Sk, torch.bfloat16, seed=1).reshape(-1).cuda()
    x = buf[8:].view(2, 1, 3, Sk)  # 16-byte offset
    assert x.data_ptr() % 32 == 16
    ref_in = x.cpu()
    lens = torch.tensor([512, 300], dtype=torch.int32).cuda()
    with torch.cuda.stream(s):
        ttlib.tt_softmax_masked(x, lens, 0.125, stream=s)
    s.synchronize()
    assert_close("softmax", torch.bfloat16, x, oracle.softmax_masked(ref_in, [512, 300], 0.125))
    assert (buf[:8].cpu() == W.scores(1, 1, 1, 8 + 2 * 3 * Sk, torch.bfloat16,
                                      seed=1).reshape(-1)[:8]).all()


@pytest.mark.parametrize("dtype", DT)
def test_staged_host_buffers(ttlib, dtype):
    lens = np.array([40, 17, 3], dtype=np.int32)
    x = W.scores(3, 12, 40, 40, dtype, seed=8)
    host = x.clone().pin_memory()
    hl = torch.as_tensor(lens).pin_memory()
    dev = torch.empty_like(x, device="cuda")
    dl = torch.empty(3, dtype=torch.int32, device="cuda")
    ttlib.tt_softmax_masked_staged(host, hl, dev, dl, W.SCALE_BERT)
    torch.cuda.synchronize()
    assert_close("softmax", dtype, host, oracle.softmax_masked(x, lens, W.SCALE_BERT))
    assert masked_bits_zero(host, lens)


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("chunks", [2, 3, 8])
def test_staged_overlap_host_buffers(ttlib, dtype, chunks):
    """Chunked H2D / kernel on one stream, D2H on a second (include/tt.h
    tt_softmax_masked_staged_overlap); an odd Sk and H * Sq make the 16-byte
    chunk granule several requests wide for 16-bit storage.  Run twice on the
    same device buffers: the second call must wait for the first's copies."""
    B, H, S = 7, 3, 37
    lens = np.array([37, 17, 3, 0, 37, 21, 1], dtype=np.int32)
    cs = torch.cuda.Stream()
    dev = torch.empty(B, H, S, S, dtype=dtype, device="cuda")
    dl = torch.empty(B, dtype=torch.int32, device="cuda")
    for rep in range(2):
        x = W.scores(B, H, S, S, dtype, seed=80 + rep)
        host = x.clone().pin_memory()
        hl = torch.as_tensor(lens).pin_memory()
        ttlib.tt_softmax_masked_staged_overlap(host, hl, dev, dl, W.SCALE_BERT, chunks,
                                               copy_stream=cs)
        torch.cuda.current_stream().synchronize()  # the contract: `stream` covers the D2H
        assert_close("softmax", dtype, host, oracle.softmax_masked(x, lens, W.SCALE_BERT),
                     f"overlap chunks={chunks} rep={rep}")
        assert masked_bits_zero(host, lens)


def test_binding_rejects_bad_tensors(ttlib):
    x = torch.zeros(2, 2, 2, 8, device="cuda")
    with pytest.raises(ValueError):
        ttlib.tt_softmax_masked(x, torch.zeros(2, dtype=torch.int64, device="cuda"), 1.0)
    with pytest.raises(ValueError):
        ttlib.tt_softmax_masked(x.transpose(2, 3), torch.zeros(2, dtype=torch.int32,
                                                                device="cuda"), 1.0)
    with pytest.raises(ttlib.TTError):
        ttlib.tt_softmax_masked(x, torch.zeros(2, dtype=torch.int32, device="cuda"),
                                float("inf"))


@pytest.mark.parametrize("dtype", DT)
def test_every_compiled_tier(ttlib, dtype):
    """Force each tier (include/tt_tune.h) and check it on shapes it can serve."""
    names = ttlib.tiers("softmax", dtype)
    try:
        for i, name in enumerate(names):
            ttlib.force_tier("softmax", dtype, i)
            for Sk in (3, 37, 130, 512, 1000, 2100, 9000):
                if ttlib.softmax_plan(dtype, 1, 1, 1, Sk) != name:
                    continue
                lens = [Sk, max(1, Sk - 5), 1, 0, Sk // 2]
                x = W.scores(len(lens), 2, 3, Sk, dtype, seed=Sk + i)
                _full_check(ttlib, x, lens, W.SCALE_BERT, f"{name} Sk={Sk}")
    finally:
        ttlib.force_tier("softmax", dtype, -1)


@pytest.mark.parametrize("dtype", DT)
def test_cluster_tier_segments_and_masks(ttlib, dtype):
    """Rows split over a thread-block cluster (softmax_cluster: one 16 384-key
    segment per CTA, (max, sum) merged through distributed shared memory):
    valid lengths ending inside each segment, on a segment boundary, in the
    first segment only (later CTAs hold only padding), 0 and 1; odd pitch so
    segments start unaligned; poison in the padding; negative scale."""
    W = 16384
    Sk = 3 * W + 5
    lens = [Sk, 1, 0, W, W + 1, 2 * W - 3, 3 * W, Sk - 1, 17]
    x = W_.scores(len(lens), 1, 1, Sk, dtype, seed=5)
    assert ttlib.softmax_plan(dtype, len(lens), 1, 1, Sk).startswith("softmax_cluster<")
    _full_check(ttlib, x, lens, W_.SCALE_BERT, "cluster")
    _full_check(ttlib, W_.poison_masked(x, lens), lens, -0.25, "cluster poison")
