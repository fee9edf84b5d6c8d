"""ctypes binding of libutf8v_cuda.so (include/utf8v_cuda.h, include/utf8v_gen.h).

The library is built in-tree by `_build.py`.  There is no fallback: if the
shared object is missing or a CUDA device is absent, calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libutf8v_cuda.so"

UTF8V_OK = 0
UTF8V_ERR_CUDA = 1
UTF8V_ERR_ARG = 2
UTF8V_ERR_NO_DEVICE = 3
UTF8V_ERR_NCCL = 4
WIDTH = 64
COMM_ID_BYTES = 128
P2P_HANDLE_BYTES = 64

_u8p = C.POINTER(C.c_uint8)
_u64p = C.POINTER(C.c_uint64)
_u32p = C.POINTER(C.c_uint32)

# name -> (restype, argtypes); every symbol include/*.h declares.
SIGNATURES: dict[str, tuple] = {
    "utf8v_cuda_abi_version": (C.c_int, []),
    "utf8v_cuda_last_error": (C.c_char_p, []),
    "utf8v_cuda_last_launch_count": (C.c_int, []),
    "utf8v_cuda_serve_stats": (C.c_int, [_u64p, _u64p]),
    "utf8v_cuda_release_thread_resources": (None, []),
    "utf8v_cuda_validate": (C.c_int, [C.c_void_p, C.c_size_t, C.c_int, _u8p]),
    "utf8v_cuda_validate_verdict": (C.c_int, [C.c_void_p, C.c_size_t, C.c_int, _u8p, _u64p,
                                              C.POINTER(C.c_int)]),
    "utf8v_cuda_validate_verdict_lanes": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int,
                                                    _u8p, _u64p, C.POINTER(C.c_int)]),
    "utf8v_cuda_validate_batch": (C.c_int, [C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t, C.c_int,
                                            C.c_void_p]),
    "utf8v_cuda_classify_lanes": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "utf8v_cuda_length_error_lanes": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "utf8v_cuda_incomplete_lanes": (C.c_int, [C.c_void_p, C.c_void_p]),
    "utf8v_cuda_ops_self_test": (C.c_int, [C.c_uint64, C.POINTER(C.c_int)]),
    "utf8v_cuda_validate_lanes_async": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64,
                                                  C.c_void_p, C.c_void_p]),
    "utf8v_cuda_validate_lanes": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int,
                                            C.POINTER(C.c_uint32)]),
    "utf8v_cuda_validate_batch_async": (C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64,
                                                  C.c_void_p, C.c_void_p]),
    "utf8v_cuda_validate_sharded": (C.c_int, [C.c_void_p, C.c_size_t, C.c_int, C.c_int, _u8p]),
    "utf8v_state_combine": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "utf8v_state_valid": (C.c_int, [C.c_void_p]),
    "utf8v_cuda_segment_state": (C.c_int, [C.c_void_p, C.c_size_t, C.c_int, C.c_void_p]),
    "utf8v_cuda_batch_states_async": (C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, C.c_void_p,
                                                C.c_void_p]),
    "utf8v_cuda_batch_states": (C.c_int, [C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p]),
    "utf8v_cuda_states_reduce_async": (C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p]),
    "utf8v_cuda_comm_unique_id": (C.c_int, [C.c_void_p]),
    "utf8v_cuda_comm_init_rank": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "utf8v_cuda_comm_init_all": (C.c_int, [C.c_int, C.c_void_p, C.c_void_p]),
    "utf8v_cuda_comm_destroy": (None, [C.c_void_p]),
    "utf8v_cuda_validate_shard_allreduce_async": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64,
                                                            C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p]),
    "utf8v_cuda_validate_shard_allreduce": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64,
                                                      C.c_int, _u8p]),
    "utf8v_cuda_verdict_shard_allreduce": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64,
                                                     C.c_uint64, C.c_int, _u8p, _u64p, C.POINTER(C.c_int)]),
    "utf8v_cuda_validate_sharded_device": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                                     C.c_void_p, _u8p]),
    "utf8v_cuda_p2p_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_void_p]),
    "utf8v_cuda_p2p_connect": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int]),
    "utf8v_cuda_p2p_validate_async": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64,
                                                C.c_void_p]),
    "utf8v_cuda_p2p_flag": (C.c_void_p, [C.c_void_p]),
    "utf8v_cuda_p2p_read": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint32)]),
    "utf8v_cuda_p2p_reset": (C.c_int, [C.c_void_p]),
    "utf8v_cuda_p2p_destroy": (None, [C.c_void_p]),
    "utf8v_cuda_stream_create": (C.c_int, [C.POINTER(C.c_void_p)]),
    "utf8v_cuda_stream_feed": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]),
    "utf8v_cuda_stream_finish": (C.c_int, [C.c_void_p, _u8p]),
    "utf8v_cuda_stream_bytes": (C.c_uint64, [C.c_void_p]),
    "utf8v_cuda_stream_destroy": (None, [C.c_void_p]),
    "utf8v_gen_stream": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_int, C.c_void_p]),
    "utf8v_gen_stream_range": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int,
                                         C.c_void_p]),
    "utf8v_gen_stream_host": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_int, C.c_int]),
    "utf8v_gen_c2": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint64, C.c_void_p,
                               C.c_void_p, C.c_void_p]),
    "utf8v_gen_c3_offsets": (C.c_int, [C.c_uint64, C.c_uint64, C.c_double, C.c_uint64, C.c_uint64,
                                       C.c_uint64, C.c_void_p]),
    "utf8v_gen_c3": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64,
                               C.c_void_p, C.c_void_p]),
    "utf8v_gen_c4": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_int, _u64p, C.c_void_p]),
}

_lock = threading.Lock()
_lib: C.CDLL | None = None


class CudaBackendError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"utf8v cuda backend status {status}: {message}")
        self.status = status


def load() -> C.CDLL:
    """Load (once) and type the shared library.  Raises if it is missing."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                    "(there is no CPU fallback)")
            lib = C.CDLL(str(LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
        return _lib


def check(status: int) -> None:
    if status != UTF8V_OK:
        msg = load().utf8v_cuda_last_error().decode(errors="replace")
        raise CudaBackendError(status, msg)
