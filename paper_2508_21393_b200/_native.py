"""ctypes binding of the C-ABI in include/zkl_b200.h (libzkl_b200.so).

The product path has no CPU fallback: if the shared library is missing or no
CUDA device is present, every prover entry point raises BackendUnavailable.
"""

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ZKL_LIB") or os.path.join(HERE, "libzkl_b200.so")

ZKL_OK = 0
ZKL_ERR_CUDA = -1
ZKL_ERR_ARG = -2
ZKL_ERR_ZERO = -3
ZKL_ERR_MISSING = -4
ZKL_ERR_UNSUPPORTED = -5

MT_FIELD, MT_I16, MT_I32, MT_I64 = 0, 1, 2, 3

EXPORTS = (
    "zkl_abi_version", "zkl_last_error", "zkl_elem_bytes", "zkl_to_mont", "zkl_from_mont",
    "zkl_lift", "zkl_eq_table", "zkl_fold", "zkl_axpy", "zkl_read", "zkl_dot",
    "zkl_sumcheck_round", "zkl_sumcheck_finish", "zkl_batch_inverse", "zkl_multiplicities",
    "zkl_matvec", "zkl_expand", "zkl_lift_u32", "zkl_launch_count", "zkl_sumcheck_prove",
    "zkl_shake256", "zkl_transcript_append", "zkl_transcript_challenge", "zkl_matmul_prove",
    "zkl_prof_enable", "zkl_prof_collect", "zkl_pair_combine", "zkl_logup_tiled_rounds",
    "zkl_multiplicities_index", "zkl_gather", "zkl_pair_multiplicities",
    "zkl_range_multiplicities", "zkl_rescale_witness", "zkl_transcript_append_ints", "zkl_transcript_challenge_vector",
    "zkl_sumcheck_prove_sharded", "zkl_shard_open", "zkl_shard_close", "zkl_shard_world",
    "zkl_shard_exchange", "zkl_igemm_i16", "zkl_matmul_prove_batch", "zkl_split_i16",
    "zkl_igemm_combine", "zkl_commit_table_bytes", "zkl_commit_tables", "zkl_commit_rows",
)


class BackendUnavailable(RuntimeError):
    """The CUDA backend (libzkl_b200.so + a CUDA device) is not available."""


class NativeError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__("zkl error %d: %s" % (code, msg))
        self.code = code


_lib = None

_vp, _u64, _i32, _i64p, _u8p = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, \
    ctypes.POINTER(ctypes.c_int64), ctypes.c_char_p

_SIGS = {
    "zkl_abi_version": ([], ctypes.c_int),
    "zkl_launch_count": ([], ctypes.c_uint64),
    "zkl_last_error": ([], ctypes.c_char_p),
    "zkl_elem_bytes": ([_i32], ctypes.c_int),
    "zkl_to_mont": ([_i32, _vp, _vp, _u64, _vp], ctypes.c_int),
    "zkl_from_mont": ([_i32, _vp, _vp, _u64, _vp], ctypes.c_int),
    "zkl_lift": ([_i32, _i32, _vp, _vp, _u64, _vp], ctypes.c_int),
    "zkl_eq_table": ([_i32, _vp, _u8p, _i32, _vp], ctypes.c_int),
    "zkl_fold": ([_i32, _vp, _vp, _u64, _u8p, _vp], ctypes.c_int),
    "zkl_axpy": ([_i32, _vp, _vp, _u8p, _vp, _u64, _vp], ctypes.c_int),
    "zkl_expand": ([_i32, _vp, _u64, _vp, _u64, _i32, _u8p, _u8p, _vp], ctypes.c_int),
    "zkl_lift_u32": ([_i32, _vp, _vp, _u64, _vp], ctypes.c_int),
    "zkl_read": ([_i32, _vp, _vp, _u64, _vp], ctypes.c_int),
    "zkl_dot": ([_i32, _vp, _vp, _vp, _u64, _vp], ctypes.c_int),
    "zkl_sumcheck_round": (
        [_i32, _vp, _i32, _u64, _i32, _u8p, _i32, _i32, _vp, _vp, _u8p, _u8p, _u8p, _vp, _vp],
        ctypes.c_int),
    "zkl_sumcheck_finish": ([_i32, _vp, _i32, _u8p, _vp, _vp], ctypes.c_int),
    "zkl_sumcheck_prove": (
        [_i32, _vp, _i32, _i32, _i32, _i32, _vp, _vp, _u8p, _u8p, _u8p, _vp, _vp, _vp, _vp,
         _vp], ctypes.c_int),
    "zkl_shake256": ([_u8p, _u64, _vp, _u64], ctypes.c_int),
    "zkl_sumcheck_prove_sharded": (
        [_i32, _vp, _i32, _i32, _i32, _i32, _vp, _vp, _u8p, _u8p, _u8p, _vp, _vp, _vp, _vp,
         _vp], ctypes.c_int),
    "zkl_shard_open": ([ctypes.c_char_p, _i32, _i32], ctypes.c_int),
    "zkl_shard_close": ([], ctypes.c_int),
    "zkl_shard_world": ([], ctypes.c_int),
    "zkl_shard_exchange": ([_vp, _u64, _vp], ctypes.c_int),
    "zkl_igemm_i16": ([_vp, _vp, _vp, _i32, _i32, _i32, _vp], ctypes.c_int),
    "zkl_split_i16": ([_vp, _u64, _vp, _vp, _vp], ctypes.c_int),
    "zkl_commit_table_bytes": ([_i32, _i32], ctypes.c_uint64),
    "zkl_commit_tables": ([_i32, _vp, _i32, _vp, _vp], ctypes.c_int),
    "zkl_commit_rows": ([_i32, _vp, _i32, _vp, _vp, _i32, _i32, _vp, _vp], ctypes.c_int),
    "zkl_igemm_combine": ([_vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_int64, _vp, _i32, _i32, _vp],
                          ctypes.c_int),
    "zkl_transcript_append": ([_vp, _u8p, _u64, _u8p, _u64], ctypes.c_int),
    "zkl_transcript_challenge": ([_i32, _vp, _u8p, _u64, _vp], ctypes.c_int),
    "zkl_batch_inverse": ([_i32, _vp, _vp, _u64, _u8p, _i64p, _vp], ctypes.c_int),
    "zkl_multiplicities": ([_i32, _vp, _u64, _vp, _u64, _vp, _i64p, _vp], ctypes.c_int),
    "zkl_matvec": ([_i32, _i32, _vp, _u64, _u64, _i32, _vp, _vp, _vp], ctypes.c_int),
    "zkl_prof_enable": ([_i32], ctypes.c_int),
    "zkl_logup_tiled_rounds": ([_i32, _vp, _i32, _i32, _i32, _u8p, _u8p, _i32, _vp, _vp, _vp,
                                _vp],
                               ctypes.c_int),
    "zkl_multiplicities_index": ([_i32, _vp, _u64, _vp, _u64, _vp, _vp, _i64p, _vp],
                                 ctypes.c_int),
    "zkl_gather": ([_i32, _vp, _vp, _u64, _vp, _u64, _u8p, _vp], ctypes.c_int),
    "zkl_pair_multiplicities": ([_i32, _vp, _i32, _vp, _i32, _u64, ctypes.c_int64, _vp, _vp, _vp,
                                 _u64, _vp, _vp, _i64p, _vp], ctypes.c_int),
    "zkl_transcript_append_ints": ([_vp, ctypes.c_char_p, _u64, _vp, _u64, _u64], ctypes.c_int),
    "zkl_transcript_challenge_vector": ([_i32, _vp, ctypes.c_char_p, _u64, _u64, _vp],
                                        ctypes.c_int),
    "zkl_rescale_witness": ([_vp, _i32, _u64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                             ctypes.c_int64, _vp, _vp, _i64p,
                             ctypes.POINTER(ctypes.c_uint64), _vp], ctypes.c_int),
    "zkl_range_multiplicities": ([_vp, _i32, _u64, ctypes.c_int64, _u64, _vp, _vp, _i64p, _vp],
                                 ctypes.c_int),
    "zkl_pair_combine": ([_i32, _vp, _vp, _i32, _vp, _i32, _u64, _u8p, _vp], ctypes.c_int),
    "zkl_prof_collect": ([_i32, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                          ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_uint64)],
                         ctypes.c_int),
    "zkl_matmul_prove": (
        [_i32, _i32, _vp, _i32, _vp, _i32, _vp, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp],
        ctypes.c_int),
    "zkl_matmul_prove_batch": (
        [_i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp], ctypes.c_int),
}


def load(path=LIB_PATH):
    """Load the shared library (no GPU needed just to load it)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise BackendUnavailable(
            "libzkl_b200.so not built (run python -m paper_2508_21393_b200.build)")
    lib = ctypes.CDLL(path)
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def lib():
    """The loaded library, with a CUDA device required (product entry)."""
    import torch

    L = load()
    if not torch.cuda.is_available():
        raise BackendUnavailable("no CUDA device: the B200 backend has no CPU fallback")
    return L


def check(rc):
    if rc != ZKL_OK:
        raise NativeError(rc, _lib.zkl_last_error().decode(errors="replace"))
    return rc


PROF_MATVEC, PROF_PHASE, PROF_EQ = 0, 1, 2


def prof_collect(kind):
    """(ms, algorithmic bytes, units, launch groups) recorded since the last
    collect for one kernel family (zkl_prof_collect)."""
    ms, by, un = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    n = ctypes.c_uint64()
    check(lib().zkl_prof_collect(kind, ctypes.byref(ms), ctypes.byref(by), ctypes.byref(un),
                                 ctypes.byref(n)))
    return ms.value, by.value, un.value, n.value
