"""K1 (quantize-on-append) parity on the B200: pool bytes bit-exact with the
CPU oracle (codes AND fp32 scales, same rounding mode), including the
contract's edge cases."""
import numpy as np
import pytest
import torch

import oracle as O
from kvq_testutil import bf16_bits, make_kv
from paper_2605_29639_b200 import KVCacheSpec, PagedKVCache, quantize_append, unpack_pages

pytestmark = pytest.mark.gpu
DT = {"int8": O.INT8, "fp8_e4m3": O.FP8_E4M3}


# Launches of up to K1_ROWS_MAX (token, head) rows take the one-warp-per-row
# kernel, larger ones the 16-token tile kernel.  ``tile=True`` pads the call
# with skipped (-1) slots so the same content also runs through the tile kernel.
K1_ROWS_MAX = 8192


def pad_to_tile(k, v, slots, Hkv):
    extra = K1_ROWS_MAX // Hkv + 1
    z = torch.zeros((extra, Hkv, 128), dtype=k.dtype)
    return (torch.cat([k, z]), torch.cat([v, z]),
            np.concatenate([np.asarray(slots, np.int32), np.full(extra, -1, np.int32)]))


def run_both(k, v, slots, Hkv, kv_dtype, num_blocks, cuda, tile=False):
    if tile:
        k, v, slots = pad_to_tile(k, v, slots, Hkv)
    cache = PagedKVCache(KVCacheSpec(Hkv, kv_dtype=kv_dtype), num_blocks, device=cuda)
    quantize_append(cache, k.to(cuda), v.to(cuda), torch.as_tensor(slots, dtype=torch.int32, device=cuda))
    gpu = cache.pool.cpu().numpy()
    ref = np.zeros((num_blocks, Hkv, O.PAGE), dtype=np.uint8)
    O.quant_append(bf16_bits(k), bf16_bits(v), slots, DT[kv_dtype], ref)
    return gpu, ref


@pytest.mark.parametrize("kv_dtype", ["int8", "fp8_e4m3"])
@pytest.mark.parametrize("T,Hkv", [(1, 8), (37, 4), (256, 8), (1024, 8), (1025, 8), (2048, 8), (300, 1)])
def test_append_bit_exact(cuda, kv_dtype, T, Hkv):
    num_blocks = (T + 15) // 16 + 5
    rng = np.random.default_rng(T * 7 + Hkv)
    slots = rng.permutation(num_blocks * 16)[:T].astype(np.int32)
    k, v = make_kv(T, Hkv, 1, kind="k"), make_kv(T, Hkv, 2, kind="v")
    gpu, ref = run_both(k, v, slots, Hkv, kv_dtype, num_blocks, cuda)
    assert np.array_equal(gpu, ref), f"{(gpu != ref).sum()} bytes differ"
    codes, scales = unpack_pages(torch.from_numpy(gpu))
    c2, s2 = O.unpack_pool(ref)
    assert np.array_equal(codes.numpy(), c2)
    assert np.array_equal(scales.numpy().view(np.uint32), s2.view(np.uint32))


def edge_rows():
    rows = []
    r = np.zeros(128, np.float32); rows.append(r)                      # all zero -> scale 0, codes 0
    r = np.zeros(128, np.float32); r[5] = -0.0; r[6] = 1e-3; rows.append(r)
    r = np.linspace(-127.5, 127.5, 128).astype(np.float32); rows.append(r)
    r = np.full(128, 0.5, np.float32); r[0] = 127.0; r[1:6] = [0.5, 1.5, 2.5, -0.5, -2.5]; rows.append(r)
    r = np.full(128, 448.0, np.float32); r[1:8] = [1.0625, 1.1875, 464, 479.99, -500, 2**-10, 3 * 2**-11]; rows.append(r)
    r = np.full(128, 1e-39, np.float32); r[3] = 9.2e-41; rows.append(r)   # bf16 subnormals
    r = np.ones(128, np.float32); r[7] = np.nan; rows.append(r)
    r = np.ones(128, np.float32); r[9] = np.inf; rows.append(r)
    r = np.ones(128, np.float32); r[9] = -np.inf; r[10] = np.nan; rows.append(r)
    r = np.full(128, 3e38, np.float32); r[2] = -3.3e38; rows.append(r)
    rng = np.random.default_rng(5)
    for e in (-30, -8, 0, 8, 30):
        rows.append((rng.standard_normal(128) * 2.0 ** e).astype(np.float32))
    return np.stack(rows)


@pytest.mark.parametrize("tile", [False, True])
@pytest.mark.parametrize("kv_dtype", ["int8", "fp8_e4m3"])
def test_append_edge_cases(cuda, kv_dtype, tile):
    x = edge_rows()
    T = x.shape[0]
    bits = O.f32_to_bf16_bits(x)
    k = torch.from_numpy(bits.view(np.int16)).view(torch.bfloat16).reshape(T, 1, 128)
    v = torch.from_numpy(bits[::-1].copy().view(np.int16)).view(torch.bfloat16).reshape(T, 1, 128)
    slots = np.arange(T, dtype=np.int32)
    gpu, ref = run_both(k, v, slots, 1, kv_dtype, (T + 15) // 16, cuda, tile=tile)
    diff = np.nonzero(gpu != ref)
    assert diff[0].size == 0, f"mismatch at {list(zip(*diff))[:8]}: gpu {gpu[diff][:8]} ref {ref[diff][:8]}"


def test_append_strided_and_skipped(cuda):
    T, Hkv = 64, 8
    qkv = make_kv(T, 3 * Hkv, 9).reshape(T, 3 * Hkv, 128)   # fused [T, (Hq+2Hkv), d] style buffer
    k, v = qkv[:, Hkv:2 * Hkv], qkv[:, 2 * Hkv:]
    slots = np.arange(T, dtype=np.int32) + 16
    slots[::5] = -1
    cache = PagedKVCache(KVCacheSpec(Hkv), 6, device=cuda)
    qkv_d = qkv.to(cuda)
    quantize_append(cache, qkv_d[:, Hkv:2 * Hkv], qkv_d[:, 2 * Hkv:],
                    torch.as_tensor(slots, device=cuda))
    ref = np.zeros((6, Hkv, O.PAGE), dtype=np.uint8)
    O.quant_append(bf16_bits(k.contiguous()), bf16_bits(v.contiguous()), slots, O.INT8, ref)
    assert np.array_equal(cache.pool.cpu().numpy(), ref)
    assert not ref[0].any(), "block 0 must stay untouched"


@pytest.mark.parametrize("tile", [False, True])
@pytest.mark.parametrize("kv_dtype", ["int8", "fp8_e4m3"])
def test_append_whole_pages_and_mixed(cuda, kv_dtype, tile):
    """Chunked-prefill shape: runs of 16 block-aligned slots take the
    whole-page path; a misaligned run and scattered decode slots in the same
    call take the per-row path.  Bytes must match the oracle either way."""
    Hkv = 8
    num_blocks = 40
    slots = list(range(5 * 16, 9 * 16))            # 4 whole pages (blocks 5..8)
    slots += list(range(12 * 16 + 3, 14 * 16 + 3))  # 32 slots, not block-aligned
    slots += [30 * 16 + 7, 2 * 16 + 0, 33 * 16 + 15, -1, 20 * 16 + 1]
    slots += list(range(36 * 16, 36 * 16 + 13))      # partial page
    slots = np.asarray(slots, dtype=np.int32)
    T = len(slots)
    k, v = make_kv(T, Hkv, 31, kind="k"), make_kv(T, Hkv, 32, kind="v")
    gpu, ref = run_both(k, v, slots, Hkv, kv_dtype, num_blocks, cuda, tile=tile)
    assert np.array_equal(gpu, ref), f"{(gpu != ref).sum()} bytes differ"


@pytest.mark.parametrize("kv_dtype", ["int8", "fp8_e4m3"])
@pytest.mark.parametrize("aligned16", [True, False])
def test_large_append_alignments(cuda, kv_dtype, aligned16):
    """Large appends take the 16-token tile kernel when K/V rows are 16-byte
    aligned, else the one-warp-per-row kernel (the tile kernel loads 16 bytes
    per lane): bit-exact either way, with a partial head group (Hkv = 6), a
    partial last tile, whole-page tiles mixed with scattered and skipped
    tokens, and strided K/V slices of a fused buffer."""
    Hkv, nb = 6, 900
    rng = np.random.default_rng(17)
    perm = rng.permutation(nb)
    slots, used = [], 0
    for p in range(600):                 # whole pages (chunked prefill)
        slots += [int(perm[used]) * 16 + t for t in range(16)]
        used += 1
    for _ in range(150):                 # scattered decode tokens, some pairs adjacent
        blk = int(perm[used]); used += 1
        o = int(rng.integers(0, 15))
        slots += [blk * 16 + o, blk * 16 + o + 1] if rng.random() < 0.5 else [blk * 16 + o]
    slots += [-1] * 5 + [int(perm[used]) * 16 + 3]
    slots += [int(perm[used + 1]) * 16 + t for t in range(9)]   # partial last tile
    T = len(slots)
    assert T % 16 and T * Hkv > 8192
    # fused [T, Hq + 2 Hkv, 128] buffer; one extra element shifts the rows off 16 B when not aligned16
    width = 3 * Hkv * 128 + (0 if aligned16 else 4)
    buf = torch.zeros((T, width), dtype=torch.bfloat16)
    k = make_kv(T, Hkv, 41, kind="k")
    v = make_kv(T, Hkv, 42, kind="v")
    off = 0 if aligned16 else 4
    buf[:, off + Hkv * 128: off + 2 * Hkv * 128] = k.reshape(T, -1)
    buf[:, off + 2 * Hkv * 128: off + 3 * Hkv * 128] = v.reshape(T, -1)
    bd = buf.to(cuda)
    kd = bd[:, off + Hkv * 128: off + 2 * Hkv * 128].view(T, Hkv, 128)
    vd = bd[:, off + 2 * Hkv * 128: off + 3 * Hkv * 128].view(T, Hkv, 128)
    assert (kd.data_ptr() % 16 == 0) == aligned16
    cache = PagedKVCache(KVCacheSpec(Hkv, kv_dtype=kv_dtype), nb, device=cuda)
    quantize_append(cache, kd, vd, torch.as_tensor(slots, dtype=torch.int32, device=cuda))
    ref = np.zeros((nb, Hkv, O.PAGE), dtype=np.uint8)
    O.quant_append(bf16_bits(k), bf16_bits(v), np.asarray(slots, np.int32), DT[kv_dtype], ref)
    gpu = cache.pool.cpu().numpy()
    assert np.array_equal(gpu, ref), int((gpu != ref).sum())


@pytest.mark.parametrize("kv_dtype", ["int8", "fp8_e4m3"])
@pytest.mark.parametrize("Hkv", [1, 3, 8])
def test_tile_append_heads_and_unequal_strides(cuda, kv_dtype, Hkv):
    """The TMA-fed tile kernel describes K and V to the TMA as two 2-D views
    [T][Hkv * 128] with their own token strides: K and V taken from two
    buffers of different widths, 1 / 3 / 8 kv heads (one head per work unit),
    T not a multiple of 16 (the last box is zero-filled past T), whole pages
    mixed with scattered and skipped tokens -- bit-exact with the oracle."""
    rng = np.random.default_rng(100 + Hkv)
    T = K1_ROWS_MAX // Hkv + 37
    nb = T + 64                      # a scattered token takes a whole block
    perm = rng.permutation(nb)
    slots, used = [], 0
    while len(slots) < T:
        if rng.random() < 0.8:
            slots += [int(perm[used]) * 16 + t for t in range(16)]
        else:
            slots += [int(perm[used]) * 16 + int(rng.integers(0, 16)), -1]
        used += 1
    slots = np.asarray(slots[:T], np.int32)
    k, v = make_kv(T, Hkv, 51, kind="k"), make_kv(T, Hkv, 52, kind="v")
    kb = torch.zeros((T, Hkv * 128 + 64), dtype=torch.bfloat16)     # token stride Hkv*128 + 64
    vb = torch.zeros((T, 2 * Hkv * 128 + 8), dtype=torch.bfloat16)  # token stride 2*Hkv*128 + 8
    kb[:, 64:] = k.reshape(T, -1)
    vb[:, 8:8 + Hkv * 128] = v.reshape(T, -1)
    kbd, vbd = kb.to(cuda), vb.to(cuda)
    kd = kbd[:, 64:].view(T, Hkv, 128)
    vd = vbd[:, 8:8 + Hkv * 128].view(T, Hkv, 128)
    assert kd.stride(0) != vd.stride(0) and kd.data_ptr() % 16 == 0 and vd.data_ptr() % 16 == 0
    cache = PagedKVCache(KVCacheSpec(Hkv, kv_dtype=kv_dtype), nb, device=cuda)
    quantize_append(cache, kd, vd, torch.as_tensor(slots, dtype=torch.int32, device=cuda))
    ref = np.zeros((nb, Hkv, O.PAGE), dtype=np.uint8)
    O.quant_append(bf16_bits(k), bf16_bits(v), slots, DT[kv_dtype], ref)
    gpu = cache.pool.cpu().numpy()
    assert np.array_equal(gpu, ref), int((gpu != ref).sum())


def test_large_append_overlapping_rows_fall_back(cuda):
    """A token stride the TMA cannot describe (0: every token reads the same
    row) still appends, through the one-warp-per-row kernel, bit-exact."""
    Hkv, T = 8, 2048                     # 16384 (token, head) rows: tile-kernel size
    row = make_kv(1, Hkv, 61, kind="k")
    k = row.to(cuda).expand(T, Hkv, 128)
    v = make_kv(1, Hkv, 62, kind="v").to(cuda).expand(T, Hkv, 128)
    assert k.stride(0) == 0
    slots = np.arange(T, dtype=np.int32)
    nb = T // 16
    cache = PagedKVCache(KVCacheSpec(Hkv), nb, device=cuda)
    quantize_append(cache, k, v, torch.as_tensor(slots, device=cuda))
    ref = np.zeros((nb, Hkv, O.PAGE), dtype=np.uint8)
    O.quant_append(bf16_bits(k.cpu().contiguous()), bf16_bits(v.cpu().contiguous()), slots, O.INT8, ref)
    assert np.array_equal(cache.pool.cpu().numpy(), ref)


@pytest.mark.parametrize("kv_dtype", ["int8", "fp8_e4m3"])
def test_tile_append_in_cuda_graph(cuda, kv_dtype):
    """The tile kernel's TMA descriptors are kernel parameters (encoded on the
    host at launch), so a captured K1 replays against whatever the captured
    K/V buffers hold at replay time: refill them, replay, bit-exact."""
    Hkv, T = 8, 1100                                   # 8800 rows: tile kernel
    nb = T // 16 + 8
    slots = np.arange(16 * 2, 16 * 2 + T, dtype=np.int32)
    kd = torch.empty((T, Hkv, 128), dtype=torch.bfloat16, device=cuda)
    vd = torch.empty_like(kd)
    sd = torch.as_tensor(slots, device=cuda)
    cache = PagedKVCache(KVCacheSpec(Hkv, kv_dtype=kv_dtype), nb, device=cuda)
    kd.copy_(make_kv(T, Hkv, 70, kind="k").to(cuda)); vd.copy_(make_kv(T, Hkv, 71, kind="v").to(cuda))
    quantize_append(cache, kd, vd, sd)                 # warm-up (lazy init outside the capture)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        quantize_append(cache, kd, vd, sd)
    for seed in (72, 74):
        k, v = make_kv(T, Hkv, seed, kind="k"), make_kv(T, Hkv, seed + 1, kind="v")
        kd.copy_(k.to(cuda)); vd.copy_(v.to(cuda))
        cache.pool.zero_()
        g.replay()
        torch.cuda.synchronize()
        ref = np.zeros((nb, Hkv, O.PAGE), dtype=np.uint8)
        O.quant_append(bf16_bits(k), bf16_bits(v), slots, DT[kv_dtype], ref)
        assert np.array_equal(cache.pool.cpu().numpy(), ref), seed


@pytest.mark.parametrize("kv_dtype", ["int8", "fp8_e4m3"])
def test_tile_append_long_ring(cuda, kv_dtype):
    """A long append: ~110 units per CTA, so every stage of the 8-stage ring
    and every team's image buffers wrap many times (mbarrier phase flips,
    double-buffered page images reused) -- pool bytes bit-exact."""
    Hkv, T = 8, 65536 + 7
    nb = T // 16 + 300
    rng = np.random.default_rng(81)
    perm = rng.permutation(nb)
    slots, used = [], 0
    while len(slots) < T:
        if rng.random() < 0.97:
            slots += [int(perm[used]) * 16 + t for t in range(16)]
        else:
            slots += [int(perm[used]) * 16 + int(rng.integers(0, 16))]
        used += 1
    slots = np.asarray(slots[:T], np.int32)
    k, v = make_kv(T, Hkv, 82, kind="k"), make_kv(T, Hkv, 83, kind="v")
    cache = PagedKVCache(KVCacheSpec(Hkv, kv_dtype=kv_dtype), nb, device=cuda)
    quantize_append(cache, k.to(cuda), v.to(cuda), torch.as_tensor(slots, device=cuda))
    ref = np.zeros((nb, Hkv, O.PAGE), dtype=np.uint8)
    O.quant_append(bf16_bits(k), bf16_bits(v), slots, DT[kv_dtype], ref)
    gpu = cache.pool.cpu().numpy()
    assert np.array_equal(gpu, ref), int((gpu != ref).sum())
