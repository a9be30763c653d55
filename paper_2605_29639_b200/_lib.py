"""ctypes binding of libkvq.so (the C ABI in include/kvq.h).

The product path has no fallback: if the shared library is missing or the
device is not a B200 (sm_100), every op raises.  Tensors cross the boundary as
raw device pointers plus sizes, and the CUDA stream as a handle, exactly as a
non-Python host (servesim's own ctypes hook) would pass
them.
"""
from __future__ import annotations

import ctypes
from pathlib import Path

from ._build import LIB_PATH

ABI_VERSION = 5  # include/kvq.h KVQ_ABI_VERSION
KVQ_OK, KVQ_EINVAL, KVQ_EUNSUPPORTED, KVQ_ECUDA = 0, -1, -2, -3
KVQ_INT8, KVQ_FP8_E4M3 = 0, 1
KVQ_OUT_BF16, KVQ_OUT_F32 = 0, 1
KVQ_OUT_BHD, KVQ_OUT_HBD = 0, 1
KVQ_STEP_APPEND_TAIL_ONLY = 1
KVQ_STEP_FUSED_APPEND = 2
KVQ_DERR_BLOCK_ID, KVQ_DERR_SEQ_LEN, KVQ_DERR_SLOT = 1, 2, 4
HEAD_DIM = 128
BLOCK_SIZE = 16
PAGE_BYTES = 4224

_c = ctypes
_vp, _i32, _i64, _sz, _f32 = _c.c_void_p, _c.c_int32, _c.c_int64, _c.c_size_t, _c.c_float

# name -> (restype, argtypes); must match include/kvq.h one for one.
SIGNATURES = {
    "kvq_version": (_c.c_int, []),
    "kvq_last_error": (_c.c_char_p, []),
    "kvq_page_bytes": (_sz, []),
    "kvq_check_device_errors": (_c.c_int, [_vp, _c.POINTER(_c.c_uint32)]),
    "kvq_profile_next_decode": (_c.c_int, [_vp]),
    "kvq_profile_next_append": (_c.c_int, [_vp]),
    "kvq_quant_append": (_c.c_int, [_vp, _vp, _i64, _i64, _vp, _i32, _i32, _i32, _vp, _i64, _vp]),
    "kvq_decode_workspace_bytes": (_sz, [_i32, _i32, _i32, _i32]),
    "kvq_decode_pages_per_split": (_i32, [_i32, _i32, _i64, _i32]),
    "kvq_decode_pages_per_split_rows": (_i32, [_i32, _i32, _i32, _i64, _i32]),
    "kvq_decode_attn": (_c.c_int, [_vp, _i64, _vp, _i64, _vp, _i32, _vp, _i32, _i32, _i32, _i32,
                                   _f32, _i32, _vp, _sz, _vp, _i32, _i32, _vp]),
    "kvq_decode_attn_mq": (_c.c_int, [_vp, _i64, _i32, _vp, _i64, _vp, _i32, _vp, _i32, _i32, _i32,
                                      _i32, _f32, _i32, _vp, _sz, _vp, _i32, _i32, _vp]),
    "kvq_copy_blocks": (_c.c_int, [_vp, _i64, _i32, _vp, _i32, _vp]),
    "kvq_gather_blocks": (_c.c_int, [_vp, _i64, _i32, _vp, _i32, _vp, _vp]),
    "kvq_scatter_blocks": (_c.c_int, [_vp, _i64, _i32, _vp, _i32, _vp, _vp]),
    "kvq_block_hashes": (_i64, [_vp, _i64, _i32, _c.c_uint64, _vp]),
    "kvq_decode_attn_peer": (_c.c_int, [_vp, _i64, _vp, _i64, _vp, _i32, _vp, _i32, _i32, _i32, _i32,
                                        _f32, _i32, _vp, _sz, _vp, _vp]),
    "kvq_decode_step": (_c.c_int, [_vp, _vp, _i64, _i64, _vp, _i32, _vp, _i64, _vp, _i64, _vp, _i32, _vp,
                                   _i32, _i32, _i32, _i32, _f32, _i32, _vp, _sz, _vp, _i32, _i32, _vp, _i32,
                                   _vp]),
    "kvq_decode_step_mq": (_c.c_int, [_vp, _vp, _i64, _i64, _vp, _i32, _vp, _i64, _i32, _vp, _i64, _vp, _i32,
                                      _vp, _i32, _i32, _i32, _i32, _f32, _i32, _vp, _sz, _vp, _i32, _i32, _vp,
                                      _i32, _vp]),
    "kvq_pipeline_submit": (_c.c_int, [_vp]),
    "kvq_sym_alloc": (_c.c_int, [_sz, _c.POINTER(_vp), _vp]),
    "kvq_sym_open": (_c.c_int, [_vp, _c.POINTER(_vp)]),
    "kvq_sym_close": (_c.c_int, [_vp]),
    "kvq_sym_free": (_c.c_int, [_vp]),
}

MAX_PEERS = 8
PEER_CTL_BYTES = 256
IPC_HANDLE_BYTES = 64


class PipeStep(_c.Structure):
    """``kvq_pipe_step`` (include/kvq.h): one slot of the native step submitter."""
    _fields_ = [("h2d_stream", _vp), ("compute_stream", _vp), ("d2h_stream", _vp), ("graph_exec", _vp),
                ("dev_in", _vp), ("host_in", _vp), ("in_bytes", _sz), ("dev_out", _vp), ("host_out", _vp),
                ("out_bytes", _sz), ("ev_in_ready", _vp), ("ev_done", _vp), ("ev_out_done", _vp),
                ("reuse", _i32), ("reserved", _i32)]


class PeerOutDesc(_c.Structure):
    """``kvq_peer_out`` (include/kvq.h): one output slot of the fused gather."""
    _fields_ = [("n_peers", _i32), ("rank", _i32), ("head_offset", _i32), ("batch_global", _i32),
                ("seq_map", _vp), ("writers_per_use", _c.c_uint32), ("reserved", _c.c_uint32),
                ("out", _vp * MAX_PEERS), ("ctl", _vp * MAX_PEERS)]

_lib = None


class KVQError(RuntimeError):
    """A libkvq entry point returned a non-zero status."""

    def __init__(self, fn: str, status: int, message: str):
        super().__init__(f"{fn} failed ({status}): {message}")
        self.status = status


def load(path: Path | str | None = None) -> ctypes.CDLL:
    """Load libkvq.so (idempotent).  Raises if it has not been built."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    import os
    p = Path(path) if path is not None else Path(os.environ.get("KVQ_LIB_PATH", LIB_PATH))
    if not p.exists():
        raise ImportError(
            f"{p} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the kvq ops)")
    lib = ctypes.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype, fn.argtypes = res, args
    if lib.kvq_version() != ABI_VERSION:
        raise ImportError(f"libkvq ABI version {lib.kvq_version()} != {ABI_VERSION} (stale build: rebuild it)")
    if path is None:
        _lib = lib
    return lib


def check(fn: str, status: int) -> None:
    if status != KVQ_OK:
        msg = load().kvq_last_error().decode(errors="replace")
        if status == KVQ_EINVAL:
            raise ValueError(f"{fn}: {msg}")
        raise KVQError(fn, status, msg)
