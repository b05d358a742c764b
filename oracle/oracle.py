"""TEST INFRASTRUCTURE ONLY — ctypes front end for the CPU oracles.

Two interchangeable backends with one Python API:

* ``port`` — ``oracle/lib/liboracle.so``, the plain-C restatement of the
  reference algorithm (oracle/cumstream_oracle.c).
* ``ref``  — ``oracle/_ref/libcumstream_ref_v{3,4}.so``, the UNMODIFIED
  reference library compiled in place from /root/reference (oracle/Makefile)
  behind our own C shim (oracle/ref_shim.cpp).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may
import this module; the product (paper_1701_06446_b200) never does.
Tensors are numpy float64 arrays in the reference's block storage
(SymTensor::data(), /root/reference/proj/include/cumstream/symten.hpp:122),
one array per order.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

_u64 = C.c_uint64
_sz = C.c_size_t
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


class OracleError(RuntimeError):
    pass


def _cpu_has_avx512() -> bool:
    try:
        with open("/proc/cpuinfo") as f:
            txt = f.read()
        return " avx512f" in txt and " avx512dq" in txt
    except OSError:
        return False


def ref_library_path() -> str | None:
    cands = ["v4", "v3"] if _cpu_has_avx512() else ["v3"]
    for v in cands:
        p = os.path.join(HERE, "_ref", f"libcumstream_ref_{v}.so")
        if os.path.exists(p):
            return p
    return None


def port_library_path() -> str | None:
    p = os.path.join(HERE, "lib", "liboracle.so")
    return p if os.path.exists(p) else None


def _ptrs(arrays: Sequence[np.ndarray]):
    arr = (_dp * len(arrays))()
    for i, a in enumerate(arrays):
        assert a.dtype == np.float64 and a.flags.c_contiguous
        arr[i] = a.ctypes.data_as(_dp)
    return arr


def _dptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


class Oracle:
    """Same calls on either backend; names follow the reference API."""

    def __init__(self, backend: str = "port", workers: int = 1):
        self.backend = backend
        self.workers = workers
        path = port_library_path() if backend == "port" else ref_library_path()
        if path is None:
            raise OracleError(f"oracle backend {backend!r} not built (make -C oracle"
                              f"{' ref' if backend == 'ref' else ''})")
        self.path = path
        self.lib = C.CDLL(path)
        self.p = "oc_" if backend == "port" else "ref_"
        self._bind()

    def _fn(self, name, argtypes, restype=C.c_int):
        f = getattr(self.lib, self.p + name)
        f.argtypes = argtypes
        f.restype = restype
        return f

    def _bind(self):
        self._layout = self._fn("layout_size", [C.c_int, C.c_int, C.c_int, C.POINTER(_u64), C.POINTER(_u64)])
        w = [C.c_int] if self.backend == "ref" else []
        self._mseries = self._fn("moment_series", [_dp, _sz, _sz, C.c_int, C.c_int] + w + [C.POINTER(_dp)])
        self._mtensor = self._fn("moment_tensor", [_dp, _sz, _sz, C.c_int, C.c_int] + w + [_dp])
        self._mupdate = self._fn("moments_update", [C.POINTER(_dp), _sz, _dp, _dp, _sz, _sz, C.c_int, C.c_int] + w)
        if self.backend == "ref":
            self._m2c = self._fn("moms2cums", [C.POINTER(_dp), C.POINTER(_dp), _sz, C.c_int, C.c_int, C.c_int, C.c_int])
            self._report = self._fn("report", [C.POINTER(_dp), _sz, C.c_int, C.c_int, C.c_int, _u64, _dp])
        else:
            self._m2c = self._fn("moms2cums", [C.POINTER(_dp), C.POINTER(_dp), C.c_int, C.c_int, C.c_int])
            self._report = self._fn("report", [C.POINTER(_dp), _sz, C.c_int, C.c_int, C.c_int, _u64, _dp])
        self._knorm = self._fn("knorm", [_dp, C.c_int, C.c_int, C.c_int, C.c_double, _dp])
        self._nu = self._fn("nu", [C.POINTER(_dp), C.c_int, C.c_int, C.c_int, C.c_int, _dp])
        self._parts = self._fn("partitions", [C.c_int, C.c_int, _ip, _sz, C.POINTER(_sz), C.POINTER(_sz)])
        if self.backend == "ref":
            self.lib.ref_last_error.restype = C.c_char_p

    def _check(self, rc: int, what: str):
        if rc != 0:
            msg = self.lib.ref_last_error().decode() if self.backend == "ref" else ""
            raise OracleError(f"{self.backend}:{what} failed rc={rc} {msg}")

    # -- layout -----------------------------------------------------------
    def layout(self, order: int, dim: int, block: int) -> tuple[int, int]:
        st, nb = _u64(), _u64()
        self._check(self._layout(order, dim, block, C.byref(st), C.byref(nb)), "layout")
        return st.value, nb.value

    def alloc_series(self, n: int, d: int, b: int) -> list[np.ndarray]:
        return [np.zeros(self.layout(s, n, b)[0]) for s in range(1, d + 1)]

    # -- moments ----------------------------------------------------------
    def moment_series(self, x: np.ndarray, d: int, b: int) -> list[np.ndarray]:
        x = np.ascontiguousarray(x, dtype=np.float64)
        rows, n = x.shape
        out = self.alloc_series(n, d, b)
        w = [self.workers] if self.backend == "ref" else []
        self._check(self._mseries(_dptr(x), rows, n, d, b, *w, _ptrs(out)), "moment_series")
        return out

    def moment_tensor(self, x: np.ndarray, order: int, b: int) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        rows, n = x.shape
        out = np.zeros(self.layout(order, n, b)[0])
        w = [self.workers] if self.backend == "ref" else []
        self._check(self._mtensor(_dptr(x), rows, n, order, b, *w, _dptr(out)), "moment_tensor")
        return out

    def moments_update(self, m: list[np.ndarray], window_len: int, xin: np.ndarray,
                       xout: np.ndarray, b: int) -> None:
        """In place, like cumstream::moments_update (moments.hpp:62)."""
        xin = np.ascontiguousarray(xin, dtype=np.float64)
        xout = np.ascontiguousarray(xout, dtype=np.float64)
        rows, n = xin.shape
        w = [self.workers] if self.backend == "ref" else []
        self._check(self._mupdate(_ptrs(m), window_len, _dptr(xin), _dptr(xout), rows, n,
                                  len(m), b, *w), "moments_update")

    # -- cumulants / norms -----------------------------------------------------
    def moms2cums(self, m: list[np.ndarray], n: int, b: int, window_len: int = 1) -> list[np.ndarray]:
        d = len(m)
        c = [np.zeros_like(t) for t in m]
        if self.backend == "ref":
            rc = self._m2c(_ptrs(m), _ptrs(c), window_len, n, d, b, self.workers)
        else:
            rc = self._m2c(_ptrs(m), _ptrs(c), n, d, b)
        self._check(rc, "moms2cums")
        return c

    def knorm(self, t: np.ndarray, order: int, n: int, b: int, k: float = 2.0) -> float:
        out = C.c_double()
        self._check(self._knorm(_dptr(t), order, n, b, k, C.byref(out)), "knorm")
        return out.value

    def nu(self, c: list[np.ndarray], n: int, b: int, order: int) -> float:
        out = C.c_double()
        self._check(self._nu(_ptrs(c), n, len(c), b, order, C.byref(out)), "nu")
        return out.value

    def report(self, c: list[np.ndarray], n: int, b: int, window: int, window_len: int) -> dict:
        d = len(c)
        out = np.zeros(6 + max(0, d - 2))
        self._check(self._report(_ptrs(c), window_len, n, d, b, window, _dptr(out)), "report")
        rep = {"window": int(out[0]), "rows": int(out[1]), "norm_c1": out[2], "norm_c2": out[3],
               "nu": {o: out[6 + o - 3] for o in range(3, d + 1)}}
        if d >= 3:
            rep["max_abs_skewness"] = out[4]
        if d >= 4:
            rep["max_abs_kurtosis"] = out[5]
        return rep

    def partitions(self, s: int, sigma: int) -> list[list[list[int]]]:
        cap = 1 << 20
        buf = (C.c_int * cap)()
        used, count = _sz(), _sz()
        self._check(self._parts(s, sigma, buf, cap, C.byref(used), C.byref(count)), "partitions")
        out, i = [], 0
        for _ in range(count.value):
            parts, seen = [], 0
            while seen < s:
                ln = buf[i]
                parts.append([buf[i + 1 + k] for k in range(ln)])
                i += 1 + ln
                seen += ln
            out.append(parts)
        return out

    # -- exact sampled-element oracle (port only) ---------------------------
    def sample_stream_moments(self, x: np.ndarray, T: int, p: int, steps: int, s: int, top: bool,
                              idx: np.ndarray) -> np.ndarray:
        """Exact M_s at sorted canonical indices idx (count x s) after prime
        over x[:T] and `steps` updates of p rows (rows in arrival order)."""
        assert self.backend == "port"
        x = np.ascontiguousarray(x, dtype=np.float64)
        idx = np.ascontiguousarray(idx, dtype=np.int32)
        out = np.empty(idx.shape[0])
        f = self._fn("sample_stream_moments", [_dp, C.c_int, _sz, _sz, C.c_int, C.c_int, C.c_int, _ip, _sz, _dp])
        self._check(f(_dptr(x), x.shape[1], T, p, steps, s, 1 if top else 0,
                      idx.ctypes.data_as(_ip), idx.shape[0], _dptr(out)), "sample_stream_moments")
        return out

    def element_offsets(self, order: int, n: int, b: int, idx: np.ndarray) -> np.ndarray:
        """Stored offsets of sorted indices idx (count x order) in block storage."""
        assert self.backend == "port"
        idx = np.ascontiguousarray(idx, dtype=np.int32)
        out = np.empty(idx.shape[0], dtype=np.uint64)
        f = self._fn("element_offsets", [C.c_int, C.c_int, C.c_int, _ip, _sz, C.POINTER(_u64)])
        self._check(f(order, n, b, idx.ctypes.data_as(_ip), idx.shape[0], out.ctypes.data_as(C.POINTER(_u64))),
                    "element_offsets")
        return out

    def sample_cumulants(self, c_lower: Sequence[np.ndarray], n: int, b: int, s: int, idx: np.ndarray,
                         m_val: np.ndarray) -> np.ndarray:
        """Exact C_s at sorted indices from M_s's values there and C_1..C_{s-1}."""
        assert self.backend == "port"
        idx = np.ascontiguousarray(idx, dtype=np.int32)
        m_val = np.ascontiguousarray(m_val, dtype=np.float64)
        out = np.empty(idx.shape[0])
        f = self._fn("sample_cumulants", [C.POINTER(_dp), C.c_int, C.c_int, C.c_int, _ip, _dp, _sz, _dp])
        self._check(f(_ptrs(list(c_lower)), n, b, s, idx.ctypes.data_as(_ip), _dptr(m_val), idx.shape[0],
                      _dptr(out)), "sample_cumulants")
        return out


class RefStream:
    """cumstream::prime/step (stream.hpp:69,73) on the reference backend."""

    def __init__(self, oracle: Oracle, n: int, d: int, t: int, t_up: int, b: int,
                 first: np.ndarray, resync_every: int = 1000):
        assert oracle.backend == "ref"
        self.o, self.n, self.d, self.b = oracle, n, d, b
        lib = oracle.lib
        lib.ref_stream_prime.argtypes = [C.c_int, C.c_int, _sz, _sz, C.c_int, _sz, C.c_int, _dp,
                                         C.POINTER(C.c_void_p)]
        lib.ref_stream_step.argtypes = [C.c_void_p, _dp, _sz, _sz, _dp, _dp]
        lib.ref_stream_report.argtypes = [C.c_void_p, _dp]
        lib.ref_stream_moments.argtypes = [C.c_void_p, C.c_int, _dp]
        lib.ref_stream_cumulants.argtypes = [C.c_void_p, C.c_int, _dp]
        lib.ref_stream_free.argtypes = [C.c_void_p]
        lib.ref_stream_free.restype = None
        first = np.ascontiguousarray(first, dtype=np.float64)
        h = C.c_void_p()
        oracle._check(lib.ref_stream_prime(n, d, t, t_up, b, resync_every, oracle.workers,
                                           _dptr(first), C.byref(h)), "stream_prime")
        self.h = h
        self.rep = np.zeros(6 + max(0, d - 2))
        self.timing = np.zeros(2)

    def step(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        self.o._check(self.o.lib.ref_stream_step(self.h, _dptr(x), x.shape[0], x.shape[1],
                                                 _dptr(self.timing), _dptr(self.rep)), "stream_step")
        return self.rep

    def moments(self, s: int) -> np.ndarray:
        out = np.zeros(self.o.layout(s, self.n, self.b)[0])
        self.o._check(self.o.lib.ref_stream_moments(self.h, s, _dptr(out)), "stream_moments")
        return out

    def cumulants(self, s: int) -> np.ndarray:
        out = np.zeros(self.o.layout(s, self.n, self.b)[0])
        self.o._check(self.o.lib.ref_stream_cumulants(self.h, s, _dptr(out)), "stream_cumulants")
        return out

    def close(self):
        if self.h:
            self.o.lib.ref_stream_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
