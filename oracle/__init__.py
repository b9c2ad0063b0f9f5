"""fp64 CPU oracle for the VSA-OGM hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package.  The
product path (``paper_2408_09066_b200``) never imports it, and the two share
no code: the arithmetic lives in ``oracle.c`` (plain C, fp64, pthreads), this
module only marshals numpy arrays through ctypes.

Every function cites the passage it follows; see the header of ``oracle.c``.
Pins that tie the oracle to the paper and to mathematics live in
``tests/test_oracle_pins.py``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so with gcc (no fast-math: fp64 stays IEEE)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-o", tmp, _SRC,
                               "-lm", "-lpthread"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i32, i64, u64, f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
        lib.oracle_splitmix64_stream.argtypes = [u64, i64, P]
        lib.oracle_splitmix64_stream.restype = u64
        lib.oracle_theta.argtypes = [u64, i32, P, P]
        lib.oracle_theta.restype = ctypes.c_int
        lib.oracle_encode.argtypes = [i32, P, P, f64, i64, P, P, P, P, i32]
        lib.oracle_encode.restype = i64
        lib.oracle_norms.argtypes = [i32, P, P]
        lib.oracle_norms.restype = None
        lib.oracle_decode_cells.argtypes = [i32, P, P, f64, P, f64, f64, f64, i64, P, P, P, i32]
        lib.oracle_decode_cells.restype = i64
        lib.oracle_hb.argtypes = [f64]
        lib.oracle_hb.restype = f64
        lib.oracle_entropy_cells.argtypes = [i32, i32, i32, i32, i32, i32, P, i32, i32, i32,
                                             f64, f64, i64, P, P, P, P]
        lib.oracle_entropy_cells.restype = i64
        lib.oracle_entropy_hist_cells.argtypes = [i32, i32, i32, i32, i32, i32, P, i32, i32, i32,
                                                  f64, f64, i64, P, P, P, P]
        lib.oracle_entropy_hist_cells.restype = i64
        lib.oracle_quadrant_centers.argtypes = [f64, f64, f64, f64, i32, P, P]
        lib.oracle_quadrant_centers.restype = None
        lib.oracle_assign_quadrants.argtypes = [f64, f64, f64, f64, i32, i64, P, P, P]
        lib.oracle_assign_quadrants.restype = None
        lib.oracle_encode_quadrants.argtypes = [i32, P, P, f64, f64, f64, f64, f64, i32, i64, P, P, P, P, i32]
        lib.oracle_encode_quadrants.restype = i64
        lib.oracle_decode_cells_quadrants.argtypes = [i32, P, P, f64, P, f64, f64, f64, f64, i32, f64, f64, f64,
                                                      i64, P, P, P, P, i32]
        lib.oracle_decode_cells_quadrants.restype = i64
        _lib = lib
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def default_threads() -> int:
    return max(1, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count() or 1)


def splitmix64_stream(seed: int, n: int) -> np.ndarray:
    out = np.zeros(n, dtype=np.uint64)
    _load().oracle_splitmix64_stream(ctypes.c_uint64(seed), n, _p(out))
    return out


def theta(seed: int, D: int):
    """Axis phases (theta_x, theta_y), each fp64[D] uniform on (-pi, pi] (Eq. 3, L2)."""
    tx = np.zeros(D, dtype=np.float64)
    ty = np.zeros(D, dtype=np.float64)
    if _load().oracle_theta(ctypes.c_uint64(seed), D, _p(tx), _p(ty)) != 0:
        raise ValueError("D must be >= 1")
    return tx, ty


def encode(tx, ty, l, xy, labels, m=None, counts=None, nthreads=None):
    """Bundle labelled points into the two class memories (Eq. 9, Eq. 5, Alg. 1 with delta=1).

    xy: float32 [n, 2] (raw metres, no centring), labels: uint8 [n].
    Returns (m complex128 [2, D], counts int64 [2], n_invalid).  If ``m`` is
    given (complex128 [2, D]) the new points are added to it (streaming)."""
    tx = np.ascontiguousarray(tx, dtype=np.float64)
    ty = np.ascontiguousarray(ty, dtype=np.float64)
    D = tx.shape[0]
    xy = np.ascontiguousarray(xy, dtype=np.float32).reshape(-1, 2)
    labels = np.ascontiguousarray(labels, dtype=np.uint8).reshape(-1)
    assert xy.shape[0] == labels.shape[0]
    mm = np.zeros((2, D, 2), dtype=np.float64)
    if m is not None:
        mm[..., 0] = np.real(m)
        mm[..., 1] = np.imag(m)
    cnt = np.zeros(2, dtype=np.int64) if counts is None else np.array(counts, dtype=np.int64)
    bad = _load().oracle_encode(D, _p(tx), _p(ty), float(l), xy.shape[0], _p(xy), _p(labels),
                                _p(mm), _p(cnt), nthreads or default_threads())
    return mm[..., 0] + 1j * mm[..., 1], cnt, int(bad)


def norms(m):
    """Eq. 10 norms n_c = ||m_c||_2, c = 0 (empty), 1 (occupied)."""
    mm = np.ascontiguousarray(np.stack([np.real(m), np.imag(m)], axis=-1), dtype=np.float64)
    out = np.zeros(2, dtype=np.float64)
    _load().oracle_norms(mm.shape[1], _p(mm), _p(out))
    return out


def decode_cells(tx, ty, l, m, x0, y0, res, rows, cols, nthreads=None):
    """Signed similarity q_c (Eq. 11 with Eq. 10 normalisation) at cell centres.

    Returns q float64 [2, n] (class 0 = empty, 1 = occupied)."""
    tx = np.ascontiguousarray(tx, dtype=np.float64)
    ty = np.ascontiguousarray(ty, dtype=np.float64)
    D = tx.shape[0]
    mm = np.ascontiguousarray(np.stack([np.real(m), np.imag(m)], axis=-1), dtype=np.float64)
    rows = np.ascontiguousarray(rows, dtype=np.int32).reshape(-1)
    cols = np.ascontiguousarray(cols, dtype=np.int32).reshape(-1)
    n = rows.shape[0]
    q = np.zeros((2, n), dtype=np.float64)
    viol = _load().oracle_decode_cells(D, _p(tx), _p(ty), float(l), _p(mm), float(x0), float(y0),
                                       float(res), n, _p(rows), _p(cols), _p(q),
                                       nthreads or default_threads())
    if viol:
        raise AssertionError(f"oracle: {viol} cells with |q| > 1 (Cauchy-Schwarz violated)")
    return q


def decode_grid(tx, ty, l, m, x0, y0, res, row_begin, row_end, col_begin, col_end, nthreads=None):
    """q over the rectangle rows [row_begin, row_end) x cols [col_begin, col_end): [2, nr, nc]."""
    rr, cc = np.meshgrid(np.arange(row_begin, row_end, dtype=np.int32),
                         np.arange(col_begin, col_end, dtype=np.int32), indexing="ij")
    q = decode_cells(tx, ty, l, m, x0, y0, res, rr.ravel(), cc.ravel(), nthreads)
    return q.reshape(2, row_end - row_begin, col_end - col_begin)


def quadrant_centers(bounds, delta):
    """getQuadrantCenters() of Alg. 1: (cx, cy) fp64 [delta^2], beta = j delta + i."""
    cx = np.zeros(delta * delta)
    cy = np.zeros(delta * delta)
    _load().oracle_quadrant_centers(*map(float, bounds), delta, _p(cx), _p(cy))
    return cx, cy


def assign_quadrants(bounds, delta, x, y):
    """Alg. 1 argmin: nearest quadrant centre of each (x, y) (fp64), ties to the lowest index."""
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
    y = np.ascontiguousarray(y, dtype=np.float64).reshape(-1)
    out = np.zeros(x.shape[0], dtype=np.int32)
    _load().oracle_assign_quadrants(*map(float, bounds), delta, x.shape[0], _p(x), _p(y), _p(out))
    return out


def encode_quadrants(tx, ty, l, bounds, delta, xy, labels, nthreads=None):
    """Alg. 1 with delta quadrants per axis: m complex128 [2 delta^2, D] (slot 2 beta + psi), counts [2 delta^2]."""
    tx = np.ascontiguousarray(tx, dtype=np.float64)
    ty = np.ascontiguousarray(ty, dtype=np.float64)
    D = tx.shape[0]
    xy = np.ascontiguousarray(xy, dtype=np.float32).reshape(-1, 2)
    labels = np.ascontiguousarray(labels, dtype=np.uint8).reshape(-1)
    ns = 2 * delta * delta
    mm = np.zeros((ns, D, 2), dtype=np.float64)
    cnt = np.zeros(ns, dtype=np.int64)
    bad = _load().oracle_encode_quadrants(D, _p(tx), _p(ty), float(l), *map(float, bounds), delta, xy.shape[0],
                                          _p(xy), _p(labels), _p(mm), _p(cnt), nthreads or default_threads())
    return mm[..., 0] + 1j * mm[..., 1], cnt, int(bad)


def decode_cells_quadrants(tx, ty, l, m, bounds, delta, x0, y0, res, rows, cols, nthreads=None):
    """Eq. 11 with delta quadrants: q [2, n] from the cell's own quadrant memories, and beta [n]."""
    tx = np.ascontiguousarray(tx, dtype=np.float64)
    ty = np.ascontiguousarray(ty, dtype=np.float64)
    D = tx.shape[0]
    mm = np.ascontiguousarray(np.stack([np.real(m), np.imag(m)], axis=-1), dtype=np.float64)
    rows = np.ascontiguousarray(rows, dtype=np.int32).reshape(-1)
    cols = np.ascontiguousarray(cols, dtype=np.int32).reshape(-1)
    n = rows.shape[0]
    q = np.zeros((2, n), dtype=np.float64)
    beta = np.zeros(n, dtype=np.int32)
    viol = _load().oracle_decode_cells_quadrants(D, _p(tx), _p(ty), float(l), _p(mm), *map(float, bounds), delta,
                                                 float(x0), float(y0), float(res), n, _p(rows), _p(cols), _p(q),
                                                 _p(beta), nthreads or default_threads())
    if viol:
        raise AssertionError(f"oracle: {viol} cells with |q| > 1")
    return q, beta


def decode_grid_quadrants(tx, ty, l, m, bounds, delta, x0, y0, res, row_begin, row_end, col_begin, col_end):
    rr, cc = np.meshgrid(np.arange(row_begin, row_end, dtype=np.int32),
                         np.arange(col_begin, col_end, dtype=np.int32), indexing="ij")
    q, beta = decode_cells_quadrants(tx, ty, l, m, bounds, delta, x0, y0, res, rr.ravel(), cc.ravel())
    shape = (row_end - row_begin, col_end - col_begin)
    return q.reshape(2, *shape), beta.reshape(shape)


def hb(p: float) -> float:
    return _load().oracle_hb(float(p))


def entropy_cells(R, C, ra, rb, ca, cb, q_region, h_occ, h_emp, disk, rho_occ, rho_emp, rows, cols):
    """Alg. 2 local entropy + global difference + Eq. 12 (3-way, L14) at target cells.

    q_region: [2, rb-ra, cb-ca] q over a region of the R x C grid containing
    every clipped footprint.  Returns (S float64 [3, n] = S_occ, S_emp, S; labels uint8 [n])."""
    q_region = np.ascontiguousarray(q_region, dtype=np.float64)
    assert q_region.shape == (2, rb - ra, cb - ca)
    rows = np.ascontiguousarray(rows, dtype=np.int32).reshape(-1)
    cols = np.ascontiguousarray(cols, dtype=np.int32).reshape(-1)
    n = rows.shape[0]
    S = np.zeros((3, n), dtype=np.float64)
    lab = np.zeros(n, dtype=np.uint8)
    viol = _load().oracle_entropy_cells(R, C, ra, rb, ca, cb, _p(q_region), h_occ, h_emp, disk,
                                        float(rho_occ), float(rho_emp), n, _p(rows), _p(cols),
                                        _p(S), _p(lab))
    if viol < 0:
        raise ValueError("oracle_entropy_cells: a footprint leaves the supplied region")
    if viol:
        raise AssertionError(f"oracle: {viol} |q| > 1 values in the entropy region")
    return S, lab


def entropy_hist_cells(R, C, ra, rb, ca, cb, p_region, h_occ, h_emp, disk, rho_occ, rho_emp, rows, cols):
    """Histogram (8-bit grey-level) entropy estimator (NEXT #2) from probabilities p [2, rb-ra, cb-ca]."""
    p_region = np.ascontiguousarray(p_region, dtype=np.float64)
    assert p_region.shape == (2, rb - ra, cb - ca)
    rows = np.ascontiguousarray(rows, dtype=np.int32).reshape(-1)
    cols = np.ascontiguousarray(cols, dtype=np.int32).reshape(-1)
    n = rows.shape[0]
    S = np.zeros((3, n), dtype=np.float64)
    lab = np.zeros(n, dtype=np.uint8)
    rc = _load().oracle_entropy_hist_cells(R, C, ra, rb, ca, cb, _p(p_region), h_occ, h_emp, disk, float(rho_occ),
                                           float(rho_emp), n, _p(rows), _p(cols), _p(S), _p(lab))
    if rc < 0:
        raise ValueError("oracle_entropy_hist_cells: a footprint leaves the supplied region")
    return S, lab


def entropy_hist_grid(p, h_occ, h_emp, disk, rho_occ, rho_emp):
    _, R, C = p.shape
    rr, cc = np.meshgrid(np.arange(R, dtype=np.int32), np.arange(C, dtype=np.int32), indexing="ij")
    S, lab = entropy_hist_cells(R, C, 0, R, 0, C, p, h_occ, h_emp, disk, rho_occ, rho_emp, rr.ravel(), cc.ravel())
    return S.reshape(3, R, C), lab.reshape(R, C)


def entropy_grid(q, h_occ, h_emp, disk, rho_occ, rho_emp):
    """Entropy maps and labels over a whole R x C grid given q [2, R, C]."""
    _, R, C = q.shape
    rr, cc = np.meshgrid(np.arange(R, dtype=np.int32), np.arange(C, dtype=np.int32), indexing="ij")
    S, lab = entropy_cells(R, C, 0, R, 0, C, q, h_occ, h_emp, disk, rho_occ, rho_emp,
                           rr.ravel(), cc.ravel())
    return S.reshape(3, R, C), lab.reshape(R, C)
