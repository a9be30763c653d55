"""The C-ABI library (libkvq.so) loads and exports exactly what include/kvq.h
declares; host-only entry points and argument validation work without a GPU."""
import ctypes
import re
from pathlib import Path

import pytest

from paper_2605_29639_b200 import _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "kvq.h"


def declared_functions():
    src = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(kvq_[a-z_0-9]+)\s*\(", src, flags=re.M)


def test_header_matches_binding():
    names = declared_functions()
    assert len(names) == 24
    assert set(names) == set(_lib.SIGNATURES)


def test_library_exports_every_symbol():
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    for name in declared_functions():
        assert hasattr(lib, name), name
    L = _lib.load()
    assert L.kvq_version() == _lib.ABI_VERSION == 5 and L.kvq_page_bytes() == 4224


def test_host_only_entry_points():
    L = _lib.load()
    # split geometry: <= 128 pages ragged (512 equal-length), >= 8 pages, <= max_blocks
    assert 64 < L.kvq_decode_pages_per_split(256, 8, 70400, 513) <= 128
    assert 8 <= L.kvq_decode_pages_per_split(8, 8, 8 * 129, 129) <= 64
    assert L.kvq_decode_pages_per_split(1, 1, 3, 3) == 3
    # query rows per kv head (ABI 5): <= 8 rows is the call above; > 8 rows,
    # equal lengths, 1-8 waves: longer splits from the wave + serial-combine
    # model (148 SMs assumed without a GPU) -- C4 at P = 8 fills one wave
    # (32 sequences x 18 splits = 576 of 592 CTA slots) instead of 111 pages
    for args in ((256, 8, 70400, 513), (8, 8, 8 * 129, 129), (128, 1, 128 * 2049, 2049)):
        assert L.kvq_decode_pages_per_split_rows(args[0], args[1], 8, *args[2:]) == \
            L.kvq_decode_pages_per_split(*args)
    assert L.kvq_decode_pages_per_split(32, 1, 32 * 8193, 8193) == 111
    assert L.kvq_decode_pages_per_split_rows(32, 1, 16, 32 * 8193, 8193) == 456
    assert L.kvq_decode_pages_per_split_rows(64, 4, 16, 64 * 8193, 8193) == 507   # C4 on one GPU: unchanged
    ws = L.kvq_decode_workspace_bytes(4, 32, 8, 3)
    assert ws >= 4 * 32 * 3 * 129 * 4 + 4 * 8 * 4


def test_argument_validation_without_gpu():
    L = _lib.load()
    st = L.kvq_quant_append(None, None, 128, 128, None, 4, 0, 0, None, 1, None)
    assert st == _lib.KVQ_EINVAL and b"bad sizes" in L.kvq_last_error()
    st = L.kvq_quant_append(16, 16, 1024, 1024, 16, 4, 8, 7, 16, 1, None)
    assert st == _lib.KVQ_EUNSUPPORTED
    st = L.kvq_decode_attn(16, 4096, 16, 10, 16, 4, 16, 2, 20, 8, 0, 0.1, 0, 256, 1 << 20, 16, 0, 0, None)
    assert st == _lib.KVQ_EINVAL and b"Hq % Hkv" in L.kvq_last_error()
    assert L.kvq_copy_blocks(None, 1, 1, None, 0, None) == 0   # no-op
    # kvq_decode_step flags: unknown bits, and KVQ_STEP_FUSED_APPEND needs T == B
    step = (16, 16, 1024, 1024, 16, 3, 16, 4096, 16, 10, 16, 4, 16, 2, 32, 8, 0, 0.1, 0, 256, 1 << 20, 16, 0, 0,
            None)
    assert L.kvq_decode_step(*step, 4, None) == _lib.KVQ_EINVAL and b"unknown flags" in L.kvq_last_error()
    assert L.kvq_decode_step(*step, _lib.KVQ_STEP_FUSED_APPEND, None) == _lib.KVQ_EINVAL
    assert b"FUSED_APPEND" in L.kvq_last_error()
    with pytest.raises(ValueError):
        _lib.check("kvq_decode_attn", _lib.KVQ_EINVAL)


def test_peer_descriptor_validation_without_gpu():
    """kvq_decode_attn_peer rejects a bad kvq_peer_out before touching the device;
    the ctypes struct mirrors the C layout."""
    L = _lib.load()
    assert ctypes.sizeof(_lib.PeerOutDesc) == 4 * 4 + 8 + 4 + 4 + 2 * 8 * _lib.MAX_PEERS
    args = (16, 4096, 16, 10, 16, 4, 16, 2, 32, 8, 0, 0.1, 0, 256, 1 << 20)
    assert L.kvq_decode_attn_peer(*args, None, None) == _lib.KVQ_EINVAL
    d = _lib.PeerOutDesc()
    d.n_peers, d.rank, d.batch_global, d.writers_per_use = 1, 0, 2, 16
    assert L.kvq_decode_attn_peer(*args, ctypes.addressof(d), None) == _lib.KVQ_EINVAL
    assert b"n_peers" in L.kvq_last_error()
    d.n_peers = 2
    assert L.kvq_decode_attn_peer(*args, ctypes.addressof(d), None) == _lib.KVQ_EINVAL
    assert b"misaligned" in L.kvq_last_error()        # null peer buffers
    d.out[0], d.out[1], d.ctl[0], d.ctl[1] = 256, 512, 1024, 1040   # ctl[1] not 128-byte aligned
    assert L.kvq_decode_attn_peer(*args, ctypes.addressof(d), None) == _lib.KVQ_EINVAL
    d.ctl[1] = 1152
    d.batch_global = 1                                  # < B
    assert L.kvq_decode_attn_peer(*args, ctypes.addressof(d), None) == _lib.KVQ_EINVAL
    h = (ctypes.c_char * _lib.IPC_HANDLE_BYTES)()
    assert L.kvq_sym_alloc(0, ctypes.byref(ctypes.c_void_p()), h) == _lib.KVQ_EINVAL


def test_ops_refuse_cpu_tensors():
    import torch
    from paper_2605_29639_b200 import KVCacheSpec, PagedKVCache, quantize_append
    cache = PagedKVCache(KVCacheSpec(2), 4, device="cpu")
    k = torch.zeros((3, 2, 128), dtype=torch.bfloat16)
    with pytest.raises(ValueError, match="no CPU fallback"):
        quantize_append(cache, k, k, torch.zeros(3, dtype=torch.int32))


def test_no_device_is_a_loud_error():
    """Without a GPU the product path fails (ECUDA), it never computes on CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    L = _lib.load()
    st = L.kvq_decode_attn(16, 4096, 16, 10, 16, 4, 16, 2, 32, 8, 0, 0.1, 0, 256, 1 << 20, 16, 0, 0, None)
    assert st == _lib.KVQ_ECUDA
