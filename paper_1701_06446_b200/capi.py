"""ctypes binding of the C ABI (include/cumstream_b200.h).

This is the Python-side FFI a maintainer would add to call the B200 hot
path; tests and bench.py go through it.  There is no CPU
fallback: if the in-tree library is missing, or a compute call is made
without a CUDA device, it raises.
"""
from __future__ import annotations

import ctypes as C
import os
import re
from typing import Sequence

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CSB_LIB_PATH") or os.path.join(PKG, "lib", "libcumstream_b200.so")
HEADER = os.path.join(os.path.dirname(PKG), "include", "cumstream_b200.h")

OK, EINVAL, ERANGE, EDOMAIN, ERUNTIME = 0, 1, 2, 3, 4
MAX_ORDER = 20

_u64 = C.c_uint64
_dp = C.POINTER(C.c_double)


class CsbError(RuntimeError):
    code = ERUNTIME


class CsbInvalidArgument(CsbError, ValueError):  # std::invalid_argument
    code = EINVAL


class CsbOutOfRange(CsbError, IndexError):  # std::out_of_range
    code = ERANGE


class CsbDomainError(CsbError, ArithmeticError):  # std::domain_error
    code = EDOMAIN


_ERRS = {EINVAL: CsbInvalidArgument, ERANGE: CsbOutOfRange, EDOMAIN: CsbDomainError,
         ERUNTIME: CsbError}


class Report(C.Structure):
    _fields_ = [("window", _u64), ("rows", _u64), ("norm_c1", C.c_double),
                ("norm_c2", C.c_double), ("nu", C.c_double * MAX_ORDER), ("n_nu", C.c_int),
                ("has_skewness", C.c_int), ("has_kurtosis", C.c_int),
                ("max_abs_skewness", C.c_double), ("max_abs_kurtosis", C.c_double)]

    def as_dict(self) -> dict:
        d = {"window": int(self.window), "rows": int(self.rows), "norm_c1": self.norm_c1,
             "norm_c2": self.norm_c2, "nu": {3 + k: self.nu[k] for k in range(self.n_nu)}}
        if self.has_skewness:
            d["max_abs_skewness"] = self.max_abs_skewness
        if self.has_kurtosis:
            d["max_abs_kurtosis"] = self.max_abs_kurtosis
        return d


class StreamConfig(C.Structure):
    _fields_ = [("dim", C.c_int), ("max_order", C.c_int), ("window_len", _u64),
                ("update_len", _u64), ("block_size", C.c_int), ("resync_every", _u64),
                ("workers", C.c_int), ("shard_index", C.c_int), ("shard_count", C.c_int)]


_AllgatherFn = C.CFUNCTYPE(C.c_int, C.c_void_p, _dp, C.POINTER(_u64), C.POINTER(_u64), C.c_int, C.c_void_p)
_AllreduceFn = C.CFUNCTYPE(C.c_int, C.c_void_p, _dp, _u64, C.c_void_p)


class CommOps(C.Structure):
    _fields_ = [("ctx", C.c_void_p), ("host_staged", C.c_int), ("allgather_ranges", _AllgatherFn),
                ("allreduce_sum", _AllreduceFn)]


class StepTiming(C.Structure):
    _fields_ = [("update_s", C.c_double), ("moms2cums_s", C.c_double)]


_lib = None


def header_symbols() -> list[str]:
    """Every csb_* function the public header declares."""
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(csb_[a-z0-9_]+)\s*\(", txt)))


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise CsbError(f"{LIB_PATH} missing: run __graft_entry__.build() "
                           "(make -C paper_1701_06446_b200/csrc)")
        L = C.CDLL(LIB_PATH)
        sig = {
            "csb_version": ([], C.c_int),
            "csb_last_error": ([], C.c_char_p),
            "csb_device_count": ([], C.c_int),
            "csb_set_device": ([C.c_int], C.c_int),
            "csb_rows_read": ([], _u64),
            "csb_layout_size": ([C.c_int, C.c_int, C.c_int, C.POINTER(_u64), C.POINTER(_u64)], C.c_int),
            "csb_block_multiplicity": ([C.POINTER(C.c_int), C.c_int, C.POINTER(_u64)], C.c_int),
            "csb_series_create": ([C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)], C.c_int),
            "csb_series_destroy": ([C.c_void_p], C.c_int),
            "csb_series_copy": ([C.c_void_p, C.c_void_p], C.c_int),
            "csb_series_shape": ([C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                  C.POINTER(C.c_int), C.POINTER(_u64)], C.c_int),
            "csb_series_set_window_len": ([C.c_void_p, _u64], C.c_int),
            "csb_series_stored": ([C.c_void_p, C.c_int, C.POINTER(_u64)], C.c_int),
            "csb_series_device_ptr": ([C.c_void_p, C.c_int, C.POINTER(C.c_void_p)], C.c_int),
            "csb_series_upload": ([C.c_void_p, C.c_int, _dp, _u64], C.c_int),
            "csb_series_download": ([C.c_void_p, C.c_int, _dp, _u64], C.c_int),
            "csb_series_gather": ([C.c_void_p, C.c_int, C.POINTER(_u64), _u64, _dp], C.c_int),
            "csb_moment_series": ([C.c_void_p, _dp, _u64, _u64], C.c_int),
            "csb_moment_tensor": ([C.c_void_p, C.c_int, _dp, _u64, _u64], C.c_int),
            "csb_moments_update": ([C.c_void_p, _dp, _dp, _u64, _u64], C.c_int),
            "csb_moms2cums": ([C.c_void_p, C.c_void_p], C.c_int),
            "csb_combine": ([C.c_void_p, _u64, C.c_void_p, _u64, C.c_void_p], C.c_int),
            "csb_moment_series_dev": ([C.c_void_p, C.c_void_p, _u64, _u64], C.c_int),
            "csb_moments_update_dev": ([C.c_void_p, C.c_void_p, C.c_void_p, _u64, _u64], C.c_int),
            "csb_knorm": ([C.c_void_p, C.c_int, C.c_double, _dp], C.c_int),
            "csb_nu": ([C.c_void_p, C.c_int, _dp], C.c_int),
            "csb_window_report": ([C.c_void_p, _u64, C.POINTER(Report)], C.c_int),
            "csb_stream_prime": ([C.POINTER(StreamConfig), _dp, _u64, _u64, C.POINTER(C.c_void_p)], C.c_int),
            "csb_stream_destroy": ([C.c_void_p], C.c_int),
            "csb_stream_step": ([C.c_void_p, _dp, _u64, _u64, C.POINTER(StepTiming), C.POINTER(Report)], C.c_int),
            "csb_stream_step_dev": ([C.c_void_p, C.c_void_p, _u64, _u64, C.POINTER(StepTiming),
                                     C.POINTER(Report)], C.c_int),
            "csb_stream_report": ([C.c_void_p, C.POINTER(Report)], C.c_int),
            "csb_stream_upload": ([C.c_void_p, _dp, _u64, _u64], C.c_int),
            "csb_stream_step_uploaded": ([C.c_void_p, C.POINTER(StepTiming), C.POINTER(Report)], C.c_int),
            "csb_stream_moments": ([C.c_void_p, C.POINTER(C.c_void_p)], C.c_int),
            "csb_stream_cumulants": ([C.c_void_p, C.POINTER(C.c_void_p)], C.c_int),
            "csb_stream_window": ([C.c_void_p, C.POINTER(_u64)], C.c_int),
            "csb_stream_materialize": ([C.c_void_p, _dp, _u64], C.c_int),
            "csb_stream_norm_partials": ([C.c_void_p, C.c_int, _dp, _u64, C.POINTER(_u64)], C.c_int),
            "csb_stream_cuda_stream": ([C.c_void_p, C.POINTER(C.c_void_p)], C.c_int),
            "csb_stream_gather_shards": ([C.c_void_p], C.c_int),
            "csb_stream_use_graphs": ([C.c_void_p, C.c_int], C.c_int),
            "csb_stream_graph_replays": ([C.c_void_p, C.POINTER(_u64)], C.c_int),
            "csb_comm_unique_id": ([C.c_char_p], C.c_int),
            "csb_comm_init": ([C.c_int, C.c_int, C.c_char_p], C.c_int),
            "csb_comm_init_ops": ([C.c_int, C.c_int, C.POINTER(CommOps)], C.c_int),
            "csb_comm_destroy": ([], C.c_int),
            "csb_comm_selftest": ([_u64], C.c_int),
            "csb_shard_range": ([C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(_u64),
                                 C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64)], C.c_int),
            "csb_moments_update_shard": ([C.c_void_p, _dp, _dp, _u64, _u64, C.c_int, C.c_int], C.c_int),
            "csb_moms2cums_shard": ([C.c_void_p, C.c_void_p, C.c_int, C.c_int], C.c_int),
            "csb_launch_count": ([], _u64),
            "csb_top_kernel": ([C.c_int, C.c_int, C.c_int, C.c_char_p, _u64], C.c_int),
            "csb_profile_enable": ([C.c_int], C.c_int),
            "csb_profile_read": ([C.c_char_p, C.POINTER(C.c_double), C.POINTER(_u64)], C.c_int),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != OK:
        msg = lib().csb_last_error().decode(errors="replace")
        raise _ERRS.get(rc, CsbError)(msg)


def _dptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def layout_size(order: int, dim: int, block: int) -> tuple[int, int]:
    st, nb = _u64(), _u64()
    check(lib().csb_layout_size(order, dim, block, C.byref(st), C.byref(nb)))
    return st.value, nb.value


def rows_read() -> int:
    return int(lib().csb_rows_read())


def launch_count() -> int:
    return int(lib().csb_launch_count())


def top_kernel(dim: int, max_order: int, block: int) -> str:
    """The kernel instantiation that updates orders d and d-1 for this shape."""
    buf = C.create_string_buffer(128)
    check(lib().csb_top_kernel(dim, max_order, block, buf, 128))
    return buf.value.decode()


def profile_enable(on: bool = True) -> None:
    check(lib().csb_profile_enable(1 if on else 0))


def profile_read(tag: str) -> tuple[float, int]:
    """(total ms, launches) of one kernel tag since the last read."""
    ms, cnt = C.c_double(), _u64()
    check(lib().csb_profile_read(tag.encode(), C.byref(ms), C.byref(cnt)))
    return ms.value, cnt.value


def shard_range(max_order: int, dim: int, block: int, shard: int, count: int, which: int = 0):
    """(blk_lo, blk_hi, elem_lo, elem_hi) of a shard for order d (which=0) or d-1 (which=1)."""
    v = [_u64() for _ in range(4)]
    check(lib().csb_shard_range(max_order, dim, block, shard, count, which, *[C.byref(x) for x in v]))
    return tuple(x.value for x in v)


def _prefer_torch_nccl() -> None:
    """The library resolves NCCL at run time and reuses a copy the process
    already holds.  If PyTorch is going to be imported in this process, import
    it first: its bundled libnccl.so.2 then is the one both sides use (loading
    the system's first would leave torch's import with a mismatched NCCL)."""
    try:
        import torch  # noqa: F401
    except ImportError:
        pass


def comm_unique_id() -> bytes:
    _prefer_torch_nccl()
    buf = C.create_string_buffer(128)
    check(lib().csb_comm_unique_id(buf))
    return buf.raw


def comm_init(nranks: int, rank: int, uid: bytes) -> None:
    _prefer_torch_nccl()
    check(lib().csb_comm_init(nranks, rank, uid))


def comm_destroy() -> None:
    check(lib().csb_comm_destroy())


def comm_selftest(count: int = 4096) -> None:
    """Collective: one allgather of ranges + one allreduce, verified (raises on mismatch)."""
    check(lib().csb_comm_selftest(count))


_comm_keepalive: list = []


def comm_init_host(nranks: int, rank: int, allgather_ranges, allreduce_sum) -> None:
    """Caller-supplied collectives over HOST buffers (csb_comm_init_ops with
    host_staged = 1).  allgather_ranges(buf, off, cnt): rank r owns
    buf[off[r]:off[r]+cnt[r]] on entry, every rank holds all ranges on
    return; allreduce_sum(buf): elementwise sum over ranks, in place.  buf
    is a float64 numpy view of the engine's pinned staging buffer."""

    def ag(_ctx, buf, off, cnt, n, _stream):
        try:
            o = [int(off[i]) for i in range(n)]
            k = [int(cnt[i]) for i in range(n)]
            size = max((a + b for a, b in zip(o, k)), default=0)
            allgather_ranges(np.ctypeslib.as_array(buf, shape=(size,)), o, k)
            return 0
        except Exception:  # noqa: BLE001 -- reported through the status code
            import traceback
            traceback.print_exc()
            return 1

    def ar(_ctx, buf, count, _stream):
        try:
            allreduce_sum(np.ctypeslib.as_array(buf, shape=(int(count),)))
            return 0
        except Exception:  # noqa: BLE001
            import traceback
            traceback.print_exc()
            return 1

    ops = CommOps(None, 1, _AllgatherFn(ag), _AllreduceFn(ar))
    _comm_keepalive.append(ops)  # the library keeps the function pointers
    check(lib().csb_comm_init_ops(nranks, rank, C.byref(ops)))


def comm_init_torch(group=None) -> None:
    """Host-staged collectives over a torch.distributed process group (gloo
    on CPU): ranges by one broadcast per owner, sums by all_reduce."""
    import torch
    import torch.distributed as dist

    world, rank = dist.get_world_size(group), dist.get_rank(group)

    def allgather_ranges(buf, off, cnt):
        t = torch.from_numpy(buf)
        for r in range(world):
            if cnt[r]:
                seg = t[off[r]: off[r] + cnt[r]].clone()
                dist.broadcast(seg, src=r, group=group)
                t[off[r]: off[r] + cnt[r]] = seg

    def allreduce_sum(buf):
        t = torch.from_numpy(buf)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)

    comm_init_host(world, rank, allgather_ranges, allreduce_sum)


def _gather(h, order: int, offsets: np.ndarray) -> np.ndarray:
    off = np.ascontiguousarray(offsets, dtype=np.uint64)
    out = np.empty(off.size)
    check(lib().csb_series_gather(h, order, off.ctypes.data_as(C.POINTER(_u64)), off.size, _dptr(out)))
    return out


class Series:
    """Device-resident MomentSeries / CumulantSeries (moments.hpp:33-42)."""

    def __init__(self, dim: int, max_order: int, block: int):
        h = C.c_void_p()
        check(lib().csb_series_create(dim, max_order, block, C.byref(h)))
        self.h = h
        self.dim, self.max_order, self.block = dim, max_order, block

    def close(self):
        if getattr(self, "h", None):
            lib().csb_series_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def window_len(self) -> int:
        wl = _u64()
        check(lib().csb_series_shape(self.h, None, None, None, C.byref(wl)))
        return wl.value

    @window_len.setter
    def window_len(self, v: int):
        check(lib().csb_series_set_window_len(self.h, v))

    def stored(self, order: int) -> int:
        st = _u64()
        check(lib().csb_series_stored(self.h, order, C.byref(st)))
        return st.value

    def device_ptr(self, order: int) -> int:
        p = C.c_void_p()
        check(lib().csb_series_device_ptr(self.h, order, C.byref(p)))
        return p.value

    def upload(self, order: int, host: np.ndarray):
        host = np.ascontiguousarray(host, dtype=np.float64)
        check(lib().csb_series_upload(self.h, order, _dptr(host), host.size))

    def download(self, order: int) -> np.ndarray:
        out = np.empty(self.stored(order))
        check(lib().csb_series_download(self.h, order, _dptr(out), out.size))
        return out

    def gather(self, order: int, offsets: np.ndarray) -> np.ndarray:
        return _gather(self.h, order, offsets)

    def tensors(self) -> list[np.ndarray]:
        return [self.download(s) for s in range(1, self.max_order + 1)]

    def copy_from(self, other: "Series"):
        check(lib().csb_series_copy(self.h, other.h))


def moment_series(x: np.ndarray, max_order: int, block: int) -> Series:
    x = np.ascontiguousarray(x, dtype=np.float64)
    s = Series(x.shape[1], max_order, block)
    check(lib().csb_moment_series(s.h, _dptr(x), x.shape[0], x.shape[1]))
    return s


def moment_tensor(x: np.ndarray, order: int, block: int) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    s = Series(x.shape[1], order, block)
    check(lib().csb_moment_tensor(s.h, order, _dptr(x), x.shape[0], x.shape[1]))
    return s.download(order)


def moments_update(m: Series, incoming: np.ndarray, outgoing: np.ndarray) -> None:
    xi = np.ascontiguousarray(incoming, dtype=np.float64)
    xo = np.ascontiguousarray(outgoing, dtype=np.float64)
    if xi.shape != xo.shape:
        raise CsbInvalidArgument("moments_update: batch sizes differ")
    check(lib().csb_moments_update(m.h, _dptr(xi), _dptr(xo), xi.shape[0], xi.shape[1]))


def moments_update_shard(m: Series, incoming: np.ndarray, outgoing: np.ndarray, shard: int, count: int) -> None:
    xi = np.ascontiguousarray(incoming, dtype=np.float64)
    xo = np.ascontiguousarray(outgoing, dtype=np.float64)
    check(lib().csb_moments_update_shard(m.h, _dptr(xi), _dptr(xo), xi.shape[0], xi.shape[1], shard, count))


def moms2cums_shard(m: Series, shard: int, count: int) -> Series:
    c = Series(m.dim, m.max_order, m.block)
    check(lib().csb_moms2cums_shard(m.h, c.h, shard, count))
    return c


def moms2cums(m: Series) -> Series:
    c = Series(m.dim, m.max_order, m.block)
    check(lib().csb_moms2cums(m.h, c.h))
    return c


def combine(m1: Series, s1: int, m2: Series, s2: int) -> Series:
    out = Series(m1.dim, m1.max_order, m1.block)
    check(lib().csb_combine(m1.h, s1, m2.h, s2, out.h))
    return out


def knorm(s: Series, order: int, k: float = 2.0) -> float:
    out = C.c_double()
    check(lib().csb_knorm(s.h, order, k, C.byref(out)))
    return out.value


def nu(c: Series, d: int) -> float:
    out = C.c_double()
    check(lib().csb_nu(c.h, d, C.byref(out)))
    return out.value


def window_report(c: Series, window: int) -> dict:
    r = Report()
    check(lib().csb_window_report(c.h, window, C.byref(r)))
    return r.as_dict()


class Stream:
    """Device-resident sliding-window engine: prime / step (stream.hpp:69,73)."""

    def __init__(self, dim: int, max_order: int, window_len: int, update_len: int, block: int,
                 first: np.ndarray, resync_every: int = 1000, shard_index: int = 0,
                 shard_count: int = 1):
        self.cfg = StreamConfig(dim, max_order, window_len, update_len, block, resync_every, 0,
                                shard_index, shard_count)
        first = np.ascontiguousarray(first, dtype=np.float64)
        h = C.c_void_p()
        check(lib().csb_stream_prime(C.byref(self.cfg), _dptr(first), first.shape[0],
                                     first.shape[1] if first.ndim == 2 else 1, C.byref(h)))
        self.h = h
        self.timing = StepTiming()
        self.rep = Report()

    def close(self):
        if getattr(self, "h", None):
            lib().csb_stream_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def step(self, x: np.ndarray, report: bool = True, timing: bool = False) -> dict | None:
        """One window update from host rows (csb_stream_step); with timing,
        self.timing holds the update / moms2cums split (StepTiming)."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        check(lib().csb_stream_step(self.h, _dptr(x), x.shape[0], x.shape[1],
                                    C.byref(self.timing) if timing else None,
                                    C.byref(self.rep) if report else None))
        return self.rep.as_dict() if report else None

    def step_dev(self, x_dev_ptr: int, rows: int, cols: int, report: bool = False):
        check(lib().csb_stream_step_dev(self.h, C.c_void_p(x_dev_ptr), rows, cols, None,
                                        C.byref(self.rep) if report else None))
        return self.rep.as_dict() if report else None

    def upload(self, x: np.ndarray) -> None:
        """Start the H2D copy of the next batch (csb_stream_upload); x must
        stay unchanged until the step consuming it returns (pinned memory
        for an asynchronous copy)."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        check(lib().csb_stream_upload(self.h, _dptr(x), x.shape[0], x.shape[1]))
        self._uploads = getattr(self, "_uploads", []) + [x]

    def step_uploaded(self, report: bool = True) -> dict | None:
        """One window update on the oldest uploaded batch."""
        check(lib().csb_stream_step_uploaded(self.h, None, C.byref(self.rep) if report else None))
        self._uploads = self._uploads[1:]
        return self.rep.as_dict() if report else None

    def use_graphs(self, on: bool) -> None:
        check(lib().csb_stream_use_graphs(self.h, 1 if on else 0))

    def graph_replays(self) -> int:
        v = _u64()
        check(lib().csb_stream_graph_replays(self.h, C.byref(v)))
        return v.value

    def gather_shards(self) -> None:
        """Collective: every rank receives all blocks of M_d and C_d (tensor dumps)."""
        check(lib().csb_stream_gather_shards(self.h))

    def report(self) -> dict:
        check(lib().csb_stream_report(self.h, C.byref(self.rep)))
        return self.rep.as_dict()

    def _series(self, fn) -> list[np.ndarray]:
        p = C.c_void_p()
        check(fn(self.h, C.byref(p)))
        d = self.cfg.max_order
        out = []
        for s in range(1, d + 1):
            st = _u64()
            check(lib().csb_series_stored(p, s, C.byref(st)))
            a = np.empty(st.value)
            check(lib().csb_series_download(p, s, _dptr(a), a.size))
            out.append(a)
        return out

    def moments(self) -> list[np.ndarray]:
        return self._series(lib().csb_stream_moments)

    def _handle(self, which: str):
        p = C.c_void_p()
        check((lib().csb_stream_moments if which == "M" else lib().csb_stream_cumulants)(self.h, C.byref(p)))
        return p

    def gather(self, which: str, order: int, offsets: np.ndarray) -> np.ndarray:
        """Sampled stored elements of M_order (which="M") or C_order ("C")."""
        return _gather(self._handle(which), order, offsets)

    def download(self, which: str, order: int) -> np.ndarray:
        """One whole stored tensor, M_order (which="M") or C_order ("C")."""
        p = self._handle(which)
        st = _u64()
        check(lib().csb_series_stored(p, order, C.byref(st)))
        a = np.empty(st.value)
        check(lib().csb_series_download(p, order, _dptr(a), a.size))
        return a

    def cumulants(self) -> list[np.ndarray]:
        return self._series(lib().csb_stream_cumulants)

    @property
    def window(self) -> int:
        w = _u64()
        check(lib().csb_stream_window(self.h, C.byref(w)))
        return w.value

    def materialize(self) -> np.ndarray:
        out = np.empty((self.cfg.window_len, self.cfg.dim))
        check(lib().csb_stream_materialize(self.h, _dptr(out), out.size))
        return out

    def cuda_stream(self) -> int:
        p = C.c_void_p()
        check(lib().csb_stream_cuda_stream(self.h, C.byref(p)))
        return p.value or 0
