"""TEST INFRASTRUCTURE ONLY — ctypes front end of the CPU oracle.

Loads ``oracle/liboracle.so`` (the d<=3 restatement, blfmm_oracle.cpp) and,
when present, ``oracle/_ref/libblfmm_ref.so`` (the reference's own sources
compiled with the shim). Imported only by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, as the checker or the CPU
baseline — never by the product package.
"""
from __future__ import annotations

import ctypes as ct
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_ORC = os.path.join(HERE, "liboracle.so")
_REF = os.path.join(HERE, "_ref", "libblfmm_ref.so")

KTYPES = {"gaussian": 0, "ga": 0, "mq": 1, "multiquadric": 1, "imq": 2, "tps": 3,
          "wendland": 4, "wendlandc2": 4, "wendland31": 5}
_DEFAULT_SHAPE = {3: 2.0, 4: 0.5, 5: 0.5}  # parse_kernel_spec defaults (kernels.cpp)

_dp = ct.POINTER(ct.c_double)
_lp = ct.POINTER(ct.c_longlong)
_ip = ct.POINTER(ct.c_int)


def _ptr(a, t=_dp):
    return a.ctypes.data_as(t) if a is not None else None


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_ORC):
            build()
        _lib = ct.CDLL(_ORC)
        _lib.orc_last_error.restype = ct.c_char_p
        _lib.orc_uniform01.restype = ct.c_double
        _lib.orc_uniform01.argtypes = [ct.c_uint64, ct.c_uint64]
        _lib.orc_sum_il.restype = ct.c_longlong
    return _lib


def ref_available() -> bool:
    return os.path.exists(_REF)


def ref():
    global _ref
    if _ref is None:
        _ref = ct.CDLL(_REF)
        _ref.ref_last_error.restype = ct.c_char_p
    return _ref


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _chk(code, which="orc"):
    if code != 0:
        l = lib() if which == "orc" else ref()
        msg = (l.orc_last_error() if which == "orc" else l.ref_last_error()).decode()
        raise OracleError(code, msg)


def parse_spec(spec: str):
    name, _, param = spec.lower().partition(":")
    shape = _DEFAULT_SHAPE.get(KTYPES[name], 1.0)
    if param:
        shape = float(param.split("=", 1)[1])
    return KTYPES[name], shape


def _box(d, lo, hi):
    lo3 = np.zeros(3)
    hi3 = np.ones(3)
    if lo is not None:
        lo3[:d] = lo
    if hi is not None:
        hi3[:d] = hi
    return lo3, hi3


# ------------------------------------------------------------------ oracle
def eval_fourier(spec, xi, d):
    t, c = parse_spec(spec)
    out = ct.c_double()
    _chk(lib().orc_eval_fourier(t, ct.c_double(c), ct.c_double(xi), d, ct.byref(out)))
    return out.value


def eval_kernel(spec, r):
    t, c = parse_spec(spec)
    out = ct.c_double()
    _chk(lib().orc_eval_kernel(t, ct.c_double(c), ct.c_double(r), ct.byref(out)))
    return out.value


def cell_average(spec, d, a, b):
    t, c = parse_spec(spec)
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    out = ct.c_double()
    _chk(lib().orc_cell_average(t, ct.c_double(c), d, _ptr(a), _ptr(b), ct.byref(out)))
    return out.value


def c_table(spec, sigma, m, d):
    t, c = parse_spec(spec)
    out = np.empty(m ** d)
    _chk(lib().orc_c_table(t, ct.c_double(c), ct.c_double(sigma), m, d, _ptr(out)))
    return out


def mlfmm(x, w, spec, sigma, m, leaf, lo=None, hi=None, c_table_in=None,
          stride=1, mode=0, stencil=10):
    """Returns (values [nrhs,n] or [n], stats dict, stage_seconds[6]).
    mode 1 = scaled grids (c_table_in then holds levels 2..leaf)."""
    if mode != 0:
        with grid_mode(mode, stencil):
            return mlfmm(x, w, spec, sigma, m, leaf, lo, hi, c_table_in, stride)
    x = np.ascontiguousarray(x, dtype=np.float64)
    n, d = x.shape
    w = np.ascontiguousarray(w, dtype=np.float64)
    nrhs = 1 if w.ndim == 1 else w.shape[0]
    out = np.zeros((nrhs, n))
    lo3, hi3 = _box(d, lo, hi)
    t, c = parse_spec(spec)
    near, far, imag = ct.c_longlong(), ct.c_longlong(), ct.c_double()
    secs = np.zeros(6)
    ctab = None if c_table_in is None else np.ascontiguousarray(c_table_in, dtype=np.float64)
    _chk(lib().orc_mlfmm(d, ct.c_long(n), _ptr(x), _ptr(lo3), _ptr(hi3), t,
                         ct.c_double(c), ct.c_double(sigma), m, leaf, _ptr(ctab),
                         nrhs, _ptr(w), _ptr(out), ct.byref(near), ct.byref(far),
                         ct.byref(imag), stride, _ptr(secs)))
    stats = dict(near_pairs=near.value, far_work=far.value, max_imag_residual=imag.value)
    return (out[0] if w.ndim == 1 else out), stats, secs


def single(x, w, spec, sigma, m, level, lo=None, hi=None, c_table_in=None):
    x = np.ascontiguousarray(x, dtype=np.float64)
    n, d = x.shape
    w = np.ascontiguousarray(w, dtype=np.float64)
    out = np.zeros(n)
    lo3, hi3 = _box(d, lo, hi)
    t, c = parse_spec(spec)
    near, far, imag = ct.c_longlong(), ct.c_longlong(), ct.c_double()
    ctab = None if c_table_in is None else np.ascontiguousarray(c_table_in, dtype=np.float64)
    _chk(lib().orc_single(d, ct.c_long(n), _ptr(x), _ptr(lo3), _ptr(hi3), t,
                          ct.c_double(c), ct.c_double(sigma), m, level, _ptr(ctab),
                          _ptr(w), _ptr(out), ct.byref(near), ct.byref(far),
                          ct.byref(imag)))
    return out, dict(near_pairs=near.value, far_work=far.value,
                     max_imag_residual=imag.value)


def direct(x, w, spec, targets=None):
    x = np.ascontiguousarray(x, dtype=np.float64)
    n, d = x.shape
    w = np.ascontiguousarray(w, dtype=np.float64)
    t, c = parse_spec(spec)
    tg = None if targets is None else np.ascontiguousarray(targets, dtype=np.int64)
    nt = n if tg is None else tg.shape[0]
    out = np.zeros(nt)
    _chk(lib().orc_direct(d, ct.c_long(n), _ptr(x), t, ct.c_double(c), _ptr(w),
                          ct.c_long(nt), _ptr(tg, _lp), _ptr(out)))
    return out


def expansions(x, w, spec, sigma, m, leaf, level, kind, lo=None, hi=None,
               c_table_in=None, mode=0, stencil=10):
    if mode != 0:
        with grid_mode(mode, stencil):
            return expansions(x, w, spec, sigma, m, leaf, level, kind, lo, hi, c_table_in)
    x = np.ascontiguousarray(x, dtype=np.float64)
    n, d = x.shape
    w = np.ascontiguousarray(w, dtype=np.float64)
    lo3, hi3 = _box(d, lo, hi)
    t, c = parse_spec(spec)
    K = m ** d
    out = np.zeros((1 << (d * level)) * K * 2)
    ctab = None if c_table_in is None else np.ascontiguousarray(c_table_in, dtype=np.float64)
    _chk(lib().orc_expansions(d, ct.c_long(n), _ptr(x), _ptr(lo3), _ptr(hi3), t,
                              ct.c_double(c), ct.c_double(sigma), m, leaf, _ptr(ctab),
                              _ptr(w), level, kind, _ptr(out)))
    z = out.reshape(-1, K, 2)
    return z[..., 0] + 1j * z[..., 1]


def tree_lists(x, leaf, level, which, lo=None, hi=None):
    """which 0 neighbors, 1 interaction list, 2 leaf points -> list of arrays."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    n, d = x.shape
    lo3, hi3 = _box(d, lo, hi)
    cnt = 1 << (d * (leaf if which == 2 else level))
    counts = np.zeros(cnt, dtype=np.int32)
    _chk(lib().orc_tree_lists(d, ct.c_long(n), _ptr(x), _ptr(lo3), _ptr(hi3), leaf,
                              level, which, _ptr(counts, _ip), None))
    ids = np.zeros(int(counts.sum()), dtype=np.int64)
    _chk(lib().orc_tree_lists(d, ct.c_long(n), _ptr(x), _ptr(lo3), _ptr(hi3), leaf,
                              level, which, _ptr(counts, _ip), _ptr(ids, _lp)))
    return np.split(ids, np.cumsum(counts)[:-1])


class grid_mode:
    """Context: GridMode (0 shared, 1 scaled) + stencil_k for the oracle and
    the compiled reference (make_level_grids, mlfmm.hpp:61-63)."""

    def __init__(self, mode=0, stencil=10):
        self.mode, self.stencil = int(mode), int(stencil)

    def __enter__(self):
        lib().orc_set_grid_mode(self.mode, self.stencil)
        if ref_available():
            ref().ref_set_grid_mode(self.mode, self.stencil)
        return self

    def __exit__(self, *a):
        lib().orc_set_grid_mode(0, 10)
        if ref_available():
            ref().ref_set_grid_mode(0, 10)


class target_leaves:
    """Context: restrict the oracle's couple / L2L / L2P / near field to the
    given dense leaf ids (row-major, level ``leaf``) and their ancestors; the
    upsweep still covers every source. Values are those of the full matvec
    at the points of the selected leaves (other entries are not evaluated)."""

    def __init__(self, ids):
        self.ids = np.ascontiguousarray(np.asarray(ids, dtype=np.int64))

    def __enter__(self):
        lib().orc_set_target_leaves(ct.c_long(self.ids.size), _ptr(self.ids, _lp))
        return self

    def __exit__(self, *a):
        lib().orc_set_target_leaves(ct.c_long(0), None)


def leaf_ids(x, leaf, lo=None, hi=None):
    """Dense row-major leaf id of every point (leaf_of, geometry.cpp:254-262)."""
    x = np.asarray(x, dtype=np.float64)
    n, d = x.shape
    lo3, hi3 = _box(d, lo, hi)
    nper = 1 << leaf
    ids = np.zeros(n, dtype=np.int64)
    for k in range(d):
        side = (hi3[k] - lo3[k]) / nper
        v = ((x[:, k] - lo3[k]) / side).astype(np.int64)
        ids = ids * nper + np.clip(v, 0, nper - 1)
    return ids


def set_threads(n: int) -> int:
    """omp_set_num_threads for the oracle (returns the resulting max threads)."""
    lib().orc_set_num_threads(int(n))
    return lib().orc_get_max_threads()


def sum_il(d, leaf, level):
    return lib().orc_sum_il(d, leaf, level)


# -------------------------------------------------------------- reference
def _spec_b(spec):
    return spec.encode()


def ref_c_table(spec, sigma, m, d):
    out = np.empty(m ** d)
    _chk(ref().ref_c_table(_spec_b(spec), ct.c_double(sigma), m, d, _ptr(out)), "ref")
    return out


def ref_eval_fourier(spec, xi, d):
    out = ct.c_double()
    _chk(ref().ref_eval_fourier(_spec_b(spec), ct.c_double(xi), d, ct.byref(out)), "ref")
    return out.value


def ref_mlfmm(x, w, spec, sigma, m, leaf, lo=None, hi=None, reps=1, mode=0, stencil=10):
    if mode != 0:
        with grid_mode(mode, stencil):
            return ref_mlfmm(x, w, spec, sigma, m, leaf, lo, hi, reps)
    x = np.ascontiguousarray(x, dtype=np.float64)
    n, d = x.shape
    assert d <= 2
    w = np.ascontiguousarray(w, dtype=np.float64)
    lo3, hi3 = _box(d, lo, hi)
    out = np.zeros(n)
    near, far, imag, secs = ct.c_longlong(), ct.c_longlong(), ct.c_double(), ct.c_double()
    _chk(ref().ref_mlfmm(d, n, _ptr(x), _ptr(lo3), _ptr(hi3), _spec_b(spec),
                         ct.c_double(sigma), m, leaf, _ptr(w), _ptr(out),
                         ct.byref(near), ct.byref(far), ct.byref(imag), reps,
                         ct.byref(secs)), "ref")
    return out, dict(near_pairs=near.value, far_work=far.value,
                     max_imag_residual=imag.value, seconds=secs.value)


def ref_single(x, w, spec, sigma, m, level, lo=None, hi=None):
    x = np.ascontiguousarray(x, dtype=np.float64)
    n, d = x.shape
    w = np.ascontiguousarray(w, dtype=np.float64)
    lo3, hi3 = _box(d, lo, hi)
    out = np.zeros(n)
    near, far, imag = ct.c_longlong(), ct.c_longlong(), ct.c_double()
    _chk(ref().ref_single(d, n, _ptr(x), _ptr(lo3), _ptr(hi3), _spec_b(spec),
                          ct.c_double(sigma), m, level, _ptr(w), _ptr(out),
                          ct.byref(near), ct.byref(far), ct.byref(imag)), "ref")
    return out, dict(near_pairs=near.value, far_work=far.value,
                     max_imag_residual=imag.value)


def ref_direct(x, w, spec):
    x = np.ascontiguousarray(x, dtype=np.float64)
    n, d = x.shape
    w = np.ascontiguousarray(w, dtype=np.float64)
    out = np.zeros(n)
    near = ct.c_longlong()
    _chk(ref().ref_direct(d, n, _ptr(x), _spec_b(spec), _ptr(w), _ptr(out),
                          ct.byref(near)), "ref")
    return out, near.value


def ref_direct_bl(x, w, spec, sigma, refinement=1024, leaf=-1, lo=None, hi=None):
    """The reference's band-limited direct oracle (leaf < 0) or its hybrid
    oracle on build_tree(ps, leaf) (fmm.cpp:57-113); d = 1."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    n, d = x.shape
    w = np.ascontiguousarray(w, dtype=np.float64)
    out = np.zeros(n)
    lo = None if lo is None else np.ascontiguousarray(lo, dtype=np.float64)
    hi = None if hi is None else np.ascontiguousarray(hi, dtype=np.float64)
    _chk(ref().ref_direct_bl(d, n, _ptr(x), None if lo is None else _ptr(lo),
                             None if hi is None else _ptr(hi), _spec_b(spec), _ptr(w),
                             ct.c_double(sigma), refinement, leaf, _ptr(out)), "ref")
    return out


def ref_eval_bandlimited(spec, sigma, x, refinement=2048):
    out = ct.c_double()
    _chk(ref().ref_eval_bandlimited(_spec_b(spec), ct.c_double(sigma), ct.c_double(x),
                                    refinement, ct.byref(out)), "ref")
    return out.value


def ref_level_c_tables(spec, sigma, m, d, leaf, mode=0, stencil=10):
    """LevelGrids::factors[l].c_vals, l = 2..leaf, as [leaf-1, K]."""
    out = np.zeros((leaf - 1, m ** d))
    with grid_mode(mode, stencil):
        _chk(ref().ref_level_c_tables(_spec_b(spec), ct.c_double(sigma), m, d, leaf,
                                      _ptr(out)), "ref")
    return out


def ref_expansions(x, w, spec, sigma, m, leaf, level, kind, lo=None, hi=None, mode=0,
                   stencil=10):
    if mode != 0:
        with grid_mode(mode, stencil):
            return ref_expansions(x, w, spec, sigma, m, leaf, level, kind, lo, hi)
    x = np.ascontiguousarray(x, dtype=np.float64)
    n, d = x.shape
    w = np.ascontiguousarray(w, dtype=np.float64)
    lo3, hi3 = _box(d, lo, hi)
    K = m ** d
    out = np.zeros((1 << (d * level)) * K * 2)
    _chk(ref().ref_expansions(d, n, _ptr(x), _ptr(lo3), _ptr(hi3), _spec_b(spec),
                              ct.c_double(sigma), m, leaf, _ptr(w), level, kind,
                              _ptr(out)), "ref")
    z = out.reshape(-1, K, 2)
    return z[..., 0] + 1j * z[..., 1]


def ref_tree_lists(x, leaf, level, which, lo=None, hi=None):
    x = np.ascontiguousarray(x, dtype=np.float64)
    n, d = x.shape
    lo3, hi3 = _box(d, lo, hi)
    cnt = 1 << (d * (leaf if which == 2 else level))
    counts = np.zeros(cnt, dtype=np.int32)
    _chk(ref().ref_tree_lists(d, n, _ptr(x), _ptr(lo3), _ptr(hi3), leaf, level,
                              which, _ptr(counts, _ip), None), "ref")
    ids = np.zeros(int(counts.sum()), dtype=np.int32)
    _chk(ref().ref_tree_lists(d, n, _ptr(x), _ptr(lo3), _ptr(hi3), leaf, level,
                              which, _ptr(counts, _ip), _ptr(ids, _ip)), "ref")
    return [a.astype(np.int64) for a in np.split(ids, np.cumsum(counts)[:-1])]
