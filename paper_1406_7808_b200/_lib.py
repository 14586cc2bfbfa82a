"""ctypes binding of the C ABI in include/sr_fmg.h (argument marshalling only).

Loads the in-tree libsrfmg.so.  There is no fallback: if the library is missing or fails
to load, importing this module raises, so no solve can silently run anywhere else.
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsrfmg.so")
MAX_LEVELS = 24

SR_OK, SR_ERR_INVALID_ARGUMENT, SR_ERR_UNSUPPORTED_CONFIG = 0, 1, 2
SR_ERR_OUT_OF_MEMORY, SR_ERR_CUDA, SR_ERR_NCCL, SR_ERR_NONFINITE = 3, 4, 5, 6
SR_F64, SR_F32 = 0, 1

STATUS_NAMES = {0: "SR_OK", 1: "SR_ERR_INVALID_ARGUMENT", 2: "SR_ERR_UNSUPPORTED_CONFIG",
                3: "SR_ERR_OUT_OF_MEMORY", 4: "SR_ERR_CUDA", 5: "SR_ERR_NCCL",
                6: "SR_ERR_NONFINITE"}

# every symbol include/sr_fmg.h declares (checked by tests/test_abi.py)
EXPORTED = [
    "sr_fmg_desc_init", "sr_fmg_create", "sr_fmg_create_ex", "sr_fmg_solve",
    "sr_fmg_solve_host", "sr_fmg_set_stream", "sr_fmg_destroy", "sr_fmg_get_info",
    "sr_fmg_last_error", "sr_fmg_kernel_count", "sr_fmg_kernel_name",
    "sr_fmg_debug_level_io", "sr_fmg_debug_op", "sr_fmg_profile_select", "sr_fmg_profile_read",
    "sr_fmg_profile_ring", "sr_fmg_profile_read_slot",
    "sr_fmg_partition", "sr_fmg_nccl_unique_id", "sr_fmg_host_store_create",
    "sr_fmg_host_store_destroy", "sr_fmg_set_host_store", "sr_fmg_solve_host_async",
    "sr_fmg_synchronize", "sr_fmg_vsolve", "sr_fmg_desc_size",
]


# optional device allocator of the descriptor: void *alloc(size_t, void *ctx),
# void free(void *, void *ctx)
ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)
FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p)


class Desc(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64 * 3), ("M", ctypes.c_int32), ("seg", ctypes.c_int32),
        ("buffer", ctypes.c_int32), ("sr_levels", ctypes.c_int32),
        ("sched_A", ctypes.c_int32), ("sched_B", ctypes.c_int32), ("dtype", ctypes.c_int32),
        ("h", ctypes.c_double), ("alpha", ctypes.c_int32), ("nu1", ctypes.c_int32),
        ("nu2", ctypes.c_int32), ("cheb_lo", ctypes.c_double), ("cheb_hi", ctypes.c_double),
        ("world", ctypes.c_int32), ("rank", ctypes.c_int32), ("pgrid", ctypes.c_int32 * 3),
        ("nccl_id", ctypes.c_void_p), ("device", ctypes.c_int32), ("stream", ctypes.c_void_p),
        ("use_graph", ctypes.c_int32), ("comm", ctypes.c_int32), ("stencil", ctypes.c_int32),
        ("nl_gamma", ctypes.c_double),
        ("alloc", ALLOC_FN), ("free", FREE_FN), ("alloc_ctx", ctypes.c_void_p),
        ("dd_min", ctypes.c_int32),
        ("coarse_idle", ctypes.c_int32),
    ]


class Info(ctypes.Structure):
    _fields_ = [
        ("M", ctypes.c_int32), ("K", ctypes.c_int32), ("T", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("n_level", (ctypes.c_int64 * 3) * MAX_LEVELS),
        ("sr", ctypes.c_int32 * MAX_LEVELS),
        ("seg_level", ctypes.c_int32 * MAX_LEVELS),
        ("buffer_level", ctypes.c_int32 * MAX_LEVELS),
        ("nseg", (ctypes.c_int32 * 3) * MAX_LEVELS),
        ("storage_ext", (ctypes.c_int32 * 3) * MAX_LEVELS),
        ("storage_pitch", (ctypes.c_int64 * 3) * MAX_LEVELS),
        ("compute_cells", ctypes.c_int64 * MAX_LEVELS),
        ("visits", ctypes.c_int64 * MAX_LEVELS),
        ("workspace_bytes", ctypes.c_int64),
        ("launches_per_solve", ctypes.c_int64),
        ("alg_bytes_per_solve", ctypes.c_double),
        ("world", ctypes.c_int32), ("rank", ctypes.c_int32),
        ("block_lo", ctypes.c_int64 * 3), ("block_n", ctypes.c_int64 * 3),
        ("f_halo", ctypes.c_int32), ("f_dims", ctypes.c_int64 * 3),
        ("exchanges_per_solve", ctypes.c_int64),
        ("level_A", ctypes.c_int32),
        ("dd", ctypes.c_int32 * MAX_LEVELS),
        ("comm_calls", ctypes.c_int64 * MAX_LEVELS),
    ]


class Partition(ctypes.Structure):
    _fields_ = [
        ("world", ctypes.c_int32), ("rank", ctypes.c_int32), ("coord", ctypes.c_int32 * 3),
        ("segs_per_rank", ctypes.c_int32 * 3),
        ("block_lo", ctypes.c_int64 * 3), ("block_n", ctypes.c_int64 * 3),
        ("f_halo", ctypes.c_int32), ("f_dims", ctypes.c_int64 * 3),
        ("level_T_lo", ctypes.c_int64 * 3), ("level_T_n", ctypes.c_int64 * 3),
        ("level_A", ctypes.c_int32),
    ]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} not found: build it with `python paper_1406_7808_b200/build.py` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P, I32, I64, D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    sig = {
        "sr_fmg_desc_init": (None, [ctypes.POINTER(Desc)]),
        "sr_fmg_create": (I32, [I64, I32, I32, I32, I32, ctypes.POINTER(P)]),
        "sr_fmg_create_ex": (I32, [ctypes.POINTER(Desc), ctypes.POINTER(P)]),
        "sr_fmg_solve": (I32, [P, P, P]),
        "sr_fmg_solve_host": (I32, [P, P, P]),
        "sr_fmg_solve_host_async": (I32, [P, P, P]),
        "sr_fmg_synchronize": (I32, [P]),
        "sr_fmg_vsolve": (I32, [P, P, P, D, I32, ctypes.POINTER(I32), ctypes.POINTER(D)]),
        "sr_fmg_desc_size": (ctypes.c_size_t, []),
        "sr_fmg_set_stream": (I32, [P, P]),
        "sr_fmg_destroy": (None, [P]),
        "sr_fmg_get_info": (I32, [P, ctypes.POINTER(Info)]),
        "sr_fmg_last_error": (ctypes.c_char_p, [P]),
        "sr_fmg_kernel_count": (I32, []),
        "sr_fmg_kernel_name": (ctypes.c_char_p, [I32]),
        "sr_fmg_debug_level_io": (I32, [P, I32, I32, I32, P]),
        "sr_fmg_debug_op": (I32, [P, I32, I32, I32, P]),
        "sr_fmg_profile_select": (I32, [P, I32, I32]),
        "sr_fmg_profile_read": (I32, [P, ctypes.POINTER(D), ctypes.POINTER(D),
                                      ctypes.POINTER(I32)]),
        "sr_fmg_profile_ring": (I32, [P, I32]),
        "sr_fmg_profile_read_slot": (I32, [P, I32, ctypes.POINTER(D), ctypes.POINTER(D),
                                           ctypes.POINTER(I32)]),
        "sr_fmg_partition": (I32, [ctypes.POINTER(Desc), ctypes.POINTER(Partition)]),
        "sr_fmg_nccl_unique_id": (I32, [P]),
        "sr_fmg_host_store_create": (P, [I32]),
        "sr_fmg_host_store_destroy": (None, [P]),
        "sr_fmg_set_host_store": (I32, [P, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()
if lib.sr_fmg_desc_size() != ctypes.sizeof(Desc):
    raise ImportError(f"{LIB_PATH}: sr_fmg_desc_t is {lib.sr_fmg_desc_size()} bytes but the "
                      f"binding's Desc is {ctypes.sizeof(Desc)}: rebuild the library")


class SrError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def check(status, handle=None):
    if status != SR_OK:
        msg = lib.sr_fmg_last_error(handle)
        raise SrError(status, msg.decode() if msg else "")


def kernel_names():
    return [lib.sr_fmg_kernel_name(i).decode() for i in range(lib.sr_fmg_kernel_count())]
