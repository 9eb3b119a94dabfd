"""Thin ctypes binding of libaa (include/aa.h, include/aa_testing.h).

Argument marshalling only: every step of the AA hot path runs in libaa's CUDA
kernels.  Functions keep the C names; vector arguments may be torch CUDA float64
tensors (contiguous) or raw device addresses (int).  There is no CPU fallback:
if libaa.so is missing or cannot be loaded, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

HERE = os.path.dirname(os.path.abspath(__file__))
# AA_LIB: an alternative in-tree build of the same library (A/B measurements of kernel variants)
LIB_PATH = os.environ.get("AA_LIB") or os.path.join(HERE, "libaa.so")

MGS, ICWY, CGS2, DCGS2 = 0, 1, 2, 3
VARIANT_IDS = {"mgs": MGS, "icwy": ICWY, "cgs2": CGS2, "dcgs2": DCGS2}
OPT_DAMPING_BETA, OPT_ICWY_DELETE, OPT_DCGS2_COND, OPT_DCGS2_RSCALE = 0, 1, 2, 3
OPT_BREAKDOWN_EPS, OPT_PROFILE, OPT_N_GLOBAL, OPT_FUSED_ALLREDUCE = 4, 5, 6, 7
OPT_CONV_NORM, OPT_DETERMINISTIC = 8, 9
STATS_LOO, STATS_RESET = 1, 2
AA_OK, AA_ERR_BREAKDOWN = 0, 6
PHASES = ("qradd", "qrdelete", "lsp_rhs", "norm_check", "other")

# every symbol include/aa.h and include/aa_testing.h declare
EXPORTS = ("aa_comm_unique_id", "aa_create", "aa_create_with_comm", "aa_set_option", "aa_init", "aa_step", "aa_step_host",
           "aa_delete_oldest", "aa_stats", "aa_reset", "aa_destroy", "aa_status_string",
           "aa_test_qradd", "aa_get_small", "aa_get_q", "aa_timings", "aa_kernel_launches",
           "aa_fill_uniform", "aa_build_info", "aa_test_timeline", "aa_test_exchange")


class AAStatsC(C.Structure):
    _fields_ = [("iter", C.c_int64), ("m_i", C.c_int32), ("sync_points_last", C.c_int32),
                ("allreduce_last", C.c_int32), ("pad0", C.c_int32), ("allreduce_total", C.c_int64),
                ("logical_sync", C.c_int64 * 5), ("logical_sync_last", C.c_int64 * 5),
                ("f_norm", C.c_double), ("dx_norm", C.c_double), ("r_ratio_min", C.c_double),
                ("loo", C.c_double), ("breakdown", C.c_int32), ("breakdown_count", C.c_int32)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libaa.so not built ({LIB_PATH}); run `python -m paper_2110_09667_b200.build`")
    lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    vp, i64, i32, dbl = C.c_void_p, C.c_int64, C.c_int, C.c_double
    sig = {
        "aa_comm_unique_id": (i32, [vp]),
        "aa_create": (i32, [C.POINTER(vp), i64, i32, i32, i32, i32, vp, vp]),
        "aa_create_with_comm": (i32, [C.POINTER(vp), i64, i32, i32, i32, i32, vp, vp]),
        "aa_set_option": (i32, [vp, i32, dbl]),
        "aa_init": (i32, [vp, vp, vp, vp]),
        "aa_step": (i32, [vp, vp, vp, vp]),
        "aa_step_host": (i32, [vp, vp, vp, vp]),
        "aa_delete_oldest": (i32, [vp]),
        "aa_stats": (i32, [vp, C.POINTER(AAStatsC), i32]),
        "aa_reset": (i32, [vp]),
        "aa_destroy": (i32, [vp]),
        "aa_status_string": (C.c_char_p, [i32]),
        "aa_test_qradd": (i32, [vp, vp]),
        "aa_get_small": (i32, [vp, vp, vp, vp, vp]),
        "aa_get_q": (i32, [vp, vp]),
        "aa_timings": (i32, [vp, vp, vp, i32]),
        "aa_kernel_launches": (i64, [vp]),
        "aa_fill_uniform": (i32, [vp, i64, i64, C.c_uint64, C.c_uint64, dbl, dbl, vp]),
        "aa_build_info": (i32, [C.c_char_p, i32]),
        "aa_test_timeline": (i32, [vp, i32, vp]),
        "aa_test_exchange": (i32, [vp, i32, i32, vp, vp]),
    }
    for name, (res, args) in sig.items():
        if os.environ.get("AA_LIB") and not hasattr(lib, name):
            continue   # an older build loaded for an A/B measurement may lack newer test hooks
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = _load()


class AAError(RuntimeError):
    def __init__(self, code, where):
        super().__init__(f"{where}: {aa_status_string(code)} (status {code})")
        self.code = code


def _chk(code, where):
    if code != AA_OK:
        raise AAError(code, where)
    return code


def _ptr(t):
    """Device (or host) address of a torch tensor / numpy array / int."""
    if t is None:
        return None
    if isinstance(t, int):
        return t
    if hasattr(t, "data_ptr"):
        import torch
        assert t.dtype == torch.float64 and t.is_contiguous(), "libaa expects contiguous float64"
        return t.data_ptr()
    if hasattr(t, "ctypes"):
        return t.ctypes.data
    raise TypeError(f"cannot take the address of {type(t)}")


def _stream_ptr(stream):
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


# ------------------------------------------------------------------ C-named wrappers
def aa_status_string(code: int) -> str:
    return _lib.aa_status_string(code).decode()


def aa_comm_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _chk(_lib.aa_comm_unique_id(buf), "aa_comm_unique_id")
    return buf.raw


def aa_create(n_local: int, m: int, qr_variant, rank: int = 0, nranks: int = 1,
              unique_id: bytes | None = None, stream=None) -> int:
    v = VARIANT_IDS[qr_variant] if isinstance(qr_variant, str) else int(qr_variant)
    h = C.c_void_p()
    uid = C.create_string_buffer(unique_id, 128) if unique_id is not None else None
    _chk(_lib.aa_create(C.byref(h), n_local, m, v, rank, nranks, uid, _stream_ptr(stream)), "aa_create")
    return h.value


def aa_create_with_comm(n_local: int, m: int, qr_variant, rank: int, nranks: int, nccl_comm: int,
                        stream=None) -> int:
    v = VARIANT_IDS[qr_variant] if isinstance(qr_variant, str) else int(qr_variant)
    h = C.c_void_p()
    _chk(_lib.aa_create_with_comm(C.byref(h), n_local, m, v, rank, nranks, nccl_comm, _stream_ptr(stream)),
         "aa_create_with_comm")
    return h.value


def torch_nccl_comm(group=None) -> int:
    """ncclComm_t of a torch.distributed NCCL process group on the current device (the
    group must be initialised eagerly, e.g. init_process_group(..., device_id=...))."""
    import torch
    import torch.distributed as dist
    pg = group or dist.distributed_c10d._get_default_group()
    return pg._get_backend(torch.device("cuda", torch.cuda.current_device()))._comm_ptr()


def aa_set_option(h: int, opt: int, val: float) -> None:
    _chk(_lib.aa_set_option(h, opt, float(val)), "aa_set_option")


def aa_init(h: int, x0, gx0, x1_out) -> None:
    _chk(_lib.aa_init(h, _ptr(x0), _ptr(gx0), _ptr(x1_out)), "aa_init")


def aa_step(h: int, x_i, gx_i, x_next) -> None:
    _chk(_lib.aa_step(h, _ptr(x_i), _ptr(gx_i), _ptr(x_next)), "aa_step")


def aa_step_host(h: int, x_i, gx_i, x_next) -> None:
    _chk(_lib.aa_step_host(h, _ptr(x_i), _ptr(gx_i), _ptr(x_next)), "aa_step_host")


def aa_delete_oldest(h: int) -> None:
    _chk(_lib.aa_delete_oldest(h), "aa_delete_oldest")


@dataclass
class Stats:
    iter: int
    m_i: int
    sync_points_last: int
    allreduce_last: int
    allreduce_total: int
    logical: dict
    logical_last: dict
    f_norm: float
    dx_norm: float
    r_ratio_min: float
    loo: float
    breakdown: bool
    breakdown_count: int


def aa_stats(h: int, loo: bool = False, reset: bool = False) -> Stats:
    s = AAStatsC()
    rc = _lib.aa_stats(h, C.byref(s), (STATS_LOO if loo else 0) | (STATS_RESET if reset else 0))
    if rc not in (AA_OK, AA_ERR_BREAKDOWN):
        raise AAError(rc, "aa_stats")
    return Stats(s.iter, s.m_i, s.sync_points_last, s.allreduce_last, s.allreduce_total,
                 dict(zip(PHASES, list(s.logical_sync))), dict(zip(PHASES, list(s.logical_sync_last))),
                 s.f_norm, s.dx_norm, s.r_ratio_min, s.loo, bool(s.breakdown),
                 int(s.breakdown_count))


def aa_reset(h: int) -> None:
    _chk(_lib.aa_reset(h), "aa_reset")


def aa_destroy(h: int) -> None:
    _chk(_lib.aa_destroy(h), "aa_destroy")


def aa_test_qradd(h: int, v) -> None:
    _chk(_lib.aa_test_qradd(h, _ptr(v)), "aa_test_qradd")


def aa_get_small(h: int, m: int, mi: int):
    import numpy as np
    R = np.zeros((m, m), order="F")
    T = np.zeros((m, m), order="F")
    g = np.zeros(max(mi, 1))
    sc = np.zeros(m)
    _chk(_lib.aa_get_small(h, R.ctypes.data, T.ctypes.data, g.ctypes.data, sc.ctypes.data), "aa_get_small")
    return R, T, g[:mi], sc


def aa_get_q(h: int, out) -> None:
    _chk(_lib.aa_get_q(h, _ptr(out)), "aa_get_q")


def aa_timings(h: int, reset: bool = False):
    import numpy as np
    ms = np.zeros(5)
    cnt = np.zeros(5, dtype=np.int64)
    _chk(_lib.aa_timings(h, ms.ctypes.data, cnt.ctypes.data, 1 if reset else 0), "aa_timings")
    return ms, cnt


def aa_kernel_launches(h: int) -> int:
    return int(_lib.aa_kernel_launches(h))


def aa_fill_uniform(out, n: int, lo: float, hi: float, *, stream_id: int, seed: int = 9667,
                    offset: int = 0, stream=None) -> None:
    _chk(_lib.aa_fill_uniform(_ptr(out), n, offset, seed, stream_id, lo, hi, _stream_ptr(stream)),
         "aa_fill_uniform")


def aa_test_timeline(h: int, enable: bool = True):
    import numpy as np
    out = np.zeros(384, dtype=np.uint64)
    _chk(_lib.aa_test_timeline(h, 1 if enable else 0, out.ctypes.data), "aa_test_timeline")
    return out[:256].reshape(2, 8, 16)


def aa_test_timeline_raw(h: int):
    import numpy as np
    out = np.zeros(384, dtype=np.uint64)
    _chk(_lib.aa_test_timeline(h, 1, out.ctypes.data), "aa_test_timeline")
    return out


def aa_test_exchange(h: int, words: int, iters: int = 200):
    """(us per fused exchange, us per ncclAllReduce) of `words` fp64 words; -1 = not available."""
    uf, un = C.c_double(-1.0), C.c_double(-1.0)
    _chk(_lib.aa_test_exchange(h, words, iters, C.byref(uf), C.byref(un)), "aa_test_exchange")
    return uf.value, un.value


def aa_build_info() -> str:
    buf = C.create_string_buffer(256)
    _chk(_lib.aa_build_info(buf, 256), "aa_build_info")
    return buf.value.decode()


# AA_OPT_ICWY_DELETE values (aa.h): the paper's rebuild as its own reduction, merged into
# QRAdd's first reduction, or the reduction-free small-matrix update (variant, not in the paper)
ICWY_DELETE_MODES = {"separate": 0, "merged": 1, "small": 2}
# AA_OPT_CONV_NORM values (aa.h)
CONV_NORM_MODES = {"lagged": 0, "immediate": 1, "off": 2}


# ------------------------------------------------------------------ convenience handle
class AndersonSolver:
    """Owns one libaa handle.  Marshalling only (no arithmetic happens here)."""

    def __init__(self, n_local, m, variant="dcgs2", rank=0, nranks=1, unique_id=None, stream=None,
                 nccl_comm=None, **options):
        self.n_local, self.m = n_local, m
        if nranks > 1 and nccl_comm is not None:
            self.h = aa_create_with_comm(n_local, m, variant, rank, nranks, nccl_comm, stream)
        else:
            self.h = aa_create(n_local, m, variant, rank, nranks, unique_id, stream)
        names = {"beta": OPT_DAMPING_BETA, "icwy_merged": OPT_ICWY_DELETE, "icwy_delete": OPT_ICWY_DELETE,
                 "dcgs2_cond": OPT_DCGS2_COND,
                 "dcgs2_rscale": OPT_DCGS2_RSCALE, "breakdown_eps": OPT_BREAKDOWN_EPS,
                 "profile": OPT_PROFILE, "n_global": OPT_N_GLOBAL, "fused_allreduce": OPT_FUSED_ALLREDUCE,
                 "conv_norm": OPT_CONV_NORM, "deterministic": OPT_DETERMINISTIC}
        for k, v in options.items():
            if v is not None:
                if k == "icwy_delete" and isinstance(v, str):
                    v = ICWY_DELETE_MODES[v]
                if k == "conv_norm" and isinstance(v, str):
                    v = CONV_NORM_MODES[v]
                aa_set_option(self.h, names[k], float(v))

    def init(self, x0, gx0, x1_out):
        aa_init(self.h, x0, gx0, x1_out)

    def step(self, x_i, gx_i, x_next):
        aa_step(self.h, x_i, gx_i, x_next)

    def step_host(self, x_i, gx_i, x_next):
        aa_step_host(self.h, x_i, gx_i, x_next)

    def delete_oldest(self):
        aa_delete_oldest(self.h)

    def stats(self, loo=False, reset=False):
        return aa_stats(self.h, loo, reset)

    def reset(self):
        aa_reset(self.h)

    def close(self):
        if self.h:
            aa_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
