"""ctypes binding of the C oracle (oracle/mfseg_oracle.c) — TEST INFRASTRUCTURE ONLY."""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "libmfseg_oracle.so")
_lib = None

_dp = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i64 = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32 = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u8 = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            build()
        L = C.CDLL(_LIB)
        L.oracle_assign.argtypes = [C.c_longlong, _dp, _dp, C.c_int, _dp, _dp, _u8, _dp, _dp,
                                    np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS"),
                                    C.c_double, C.c_double, C.c_double, _i64, C.c_int]
        L.oracle_run.argtypes = [C.c_longlong, _dp, _dp, C.c_longlong, _dp, _dp, _dp, _dp,
                                 np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS"),
                                 C.c_double, C.c_double, C.c_double, C.c_double, C.c_double,
                                 C.c_int, C.c_int, _i32, _i32, _dp, _dp, _dp, _u8, _u8, _i64,
                                 _i64, _u8, C.POINTER(C.c_int), C.POINTER(C.c_int), _dp]
        L.oracle_assign_field.argtypes = [C.c_longlong, C.c_void_p, _i32, _dp, _dp, _dp, _dp,
                                          C.c_int, _dp, _dp, _u8, _dp, _dp, _i32, C.c_double,
                                          C.c_double, C.c_double, _i64, C.c_int]
        L.oracle_run_grid.argtypes = [C.c_longlong, _dp, _dp, C.c_int, _i32, _dp, _dp, _dp, _dp,
                                      _dp, _dp, _i32, C.c_double, C.c_double, C.c_double,
                                      C.c_double, C.c_double, C.c_int, C.c_int, _i32, _i32, _dp,
                                      _dp, _dp, _u8, _u8, _i64, _i64, _u8, C.POINTER(C.c_int),
                                      C.POINTER(C.c_int), _dp]
        _lib = L
    return _lib


def _f(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a.reshape(shape) if shape is not None else a


def assign(sloc, sval, cloc, cval, chas, mins, C_, k, wv, wd, cf, threads=os.cpu_count()):
    """Windowed assignment of samples (n,4) given centres; returns int64 labels."""
    sloc = _f(sloc).reshape(-1, 4)
    n = len(sloc)
    out = np.empty(n, np.int64)
    K = len(cloc)
    lib().oracle_assign(n, sloc, _f(sval), K, _f(cloc).reshape(-1, 4), _f(np.nan_to_num(cval)),
                        np.ascontiguousarray(chas, np.uint8), _f(mins), _f(C_),
                        np.ascontiguousarray(k, np.int32), float(wv), float(wd), float(cf), out,
                        int(threads))
    return out


def assign_field(dims, origin, spacing, times, values, cloc, cval, chas, mins, C_, k, wv, wd, cf,
                 idx=None, threads=os.cpu_count()):
    """Windowed assignment of field cells (flat indices `idx`, or all cells) given
    centres; cell locations are derived from the geometry (model.py:137-150)."""
    values = _f(values).reshape(-1)
    nt = len(times)
    if idx is None:
        n, ip = len(values), None
    else:
        idx = np.ascontiguousarray(idx, np.int64)
        n, ip = len(idx), idx.ctypes.data
    out = np.empty(n, np.int64)
    rc = lib().oracle_assign_field(n, ip, np.ascontiguousarray(dims, np.int32), _f(origin),
                                   _f(spacing), _f(times), values, len(cloc),
                                   _f(cloc).reshape(-1, 4), _f(np.nan_to_num(cval)),
                                   np.ascontiguousarray(chas, np.uint8), _f(mins), _f(C_),
                                   np.ascontiguousarray(k, np.int32), float(wv), float(wd),
                                   float(cf), out, int(threads))
    if rc != 0 or nt == 0 and n:
        raise RuntimeError("oracle_assign_field failed")
    return out


def _run_out(n_p, n_f, K, max_iterations):
    return {
        "point_labels": np.empty(n_p, np.int32), "field_labels": np.empty(n_f, np.int32),
        "loc": np.empty((K, 4)), "pval": np.empty(K), "fval": np.empty(K),
        "has_p": np.empty(K, np.uint8), "has_f": np.empty(K, np.uint8),
        "n_points": np.empty(K, np.int64), "n_fields": np.empty(K, np.int64),
        "dormant": np.empty(K, np.uint8), "progress": np.zeros(max(int(max_iterations), 1)),
    }


def _finish(out, rc, it, conv, what):
    if rc != 0:
        raise RuntimeError(f"{what} failed")
    out["iterations_used"], out["converged"] = it.value, bool(conv.value)
    out["progress"] = out["progress"][: it.value]
    for key in ("has_p", "has_f", "dormant"):
        out[key] = out[key].astype(bool)
    return out


def run_grid(p_loc, p_val, dims, origin, spacing, times, f_val, mins, maxs, k, c_f=1.0, w_d=1.0,
             w_p=1.0, w_f=1.0, eps_c=0.01, max_iterations=50, threads=os.cpu_count()):
    """engine.run restated in C, the field given by its geometry (no loc4 array)."""
    p_loc = _f(p_loc).reshape(-1, 4)
    p_val, f_val = _f(p_val).reshape(-1), _f(f_val).reshape(-1)
    K = int(np.prod(k))
    out = _run_out(len(p_loc), len(f_val), K, max_iterations)
    it, conv = C.c_int(0), C.c_int(0)
    rc = lib().oracle_run_grid(len(p_loc), p_loc, p_val, len(times),
                               np.ascontiguousarray(dims, np.int32), _f(origin), _f(spacing),
                               _f(times), f_val, _f(mins), _f(maxs),
                               np.ascontiguousarray(k, np.int32), c_f, w_d, w_p, w_f, eps_c,
                               int(max_iterations), int(threads), out["point_labels"],
                               out["field_labels"], out["loc"], out["pval"], out["fval"],
                               out["has_p"], out["has_f"], out["n_points"], out["n_fields"],
                               out["dormant"], C.byref(it), C.byref(conv), out["progress"])
    return _finish(out, rc, it, conv, "oracle_run_grid")


def run(p_loc, p_val, f_loc, f_val, mins, maxs, k, c_f=1.0, w_d=1.0, w_p=1.0, w_f=1.0,
        eps_c=0.01, max_iterations=50, threads=os.cpu_count()):
    """engine.run restated in C. Returns a dict of labels, state and convergence info."""
    p_loc = _f(p_loc).reshape(-1, 4)
    f_loc = _f(f_loc).reshape(-1, 4)
    p_val, f_val = _f(p_val).reshape(-1), _f(f_val).reshape(-1)
    K = int(np.prod(k))
    out = _run_out(len(p_loc), len(f_loc), K, max_iterations)
    it, conv = C.c_int(0), C.c_int(0)
    rc = lib().oracle_run(len(p_loc), p_loc, p_val, len(f_loc), f_loc, f_val, _f(mins), _f(maxs),
                          np.ascontiguousarray(k, np.int32), c_f, w_d, w_p, w_f, eps_c,
                          int(max_iterations), int(threads), out["point_labels"],
                          out["field_labels"], out["loc"], out["pval"], out["fval"],
                          out["has_p"], out["has_f"], out["n_points"], out["n_fields"],
                          out["dormant"], C.byref(it), C.byref(conv), out["progress"])
    return _finish(out, rc, it, conv, "oracle_run")
