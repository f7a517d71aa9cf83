"""Calls the BLAS kernels numpy's LAPACK uses (numpy's bundled OpenBLAS,
ILP64 symbols) so candidate summation orders can be checked against them."""
import ctypes as C
import glob
import os

import numpy as np

_lib = C.CDLL(glob.glob(os.path.join(os.path.dirname(np.__file__) + ".libs", "libscipy_openblas64_*.so"))[0])
I = C.c_int64
D = C.c_double
P = C.POINTER


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def dnrm2(x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    f = _lib.scipy_dnrm2_64_
    f.restype = D
    return f(C.byref(I(len(x))), _p(x), C.byref(I(1)))


def dgemv(trans, A, x, alpha=1.0, beta=0.0, y=None):
    """A is a 2-D array interpreted as the Fortran matrix A (m x n)."""
    Af = np.asfortranarray(A, dtype=np.float64)
    m, n = Af.shape
    x = np.ascontiguousarray(x, dtype=np.float64)
    ylen = n if trans == "T" else m
    y = np.zeros(ylen) if y is None else np.ascontiguousarray(y, dtype=np.float64).copy()
    _lib.scipy_dgemv_64_(C.c_char_p(trans.encode()), C.byref(I(m)), C.byref(I(n)), C.byref(D(alpha)), _p(Af),
                         C.byref(I(m)), _p(x), C.byref(I(1)), C.byref(D(beta)), _p(y), C.byref(I(1)), I(1))
    return y


def dger(A, x, y, alpha):
    Af = np.asfortranarray(A, dtype=np.float64).copy(order="F")
    m, n = Af.shape
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    _lib.scipy_dger_64_(C.byref(I(m)), C.byref(I(n)), C.byref(D(alpha)), _p(x), C.byref(I(1)), _p(y),
                        C.byref(I(1)), _p(Af), C.byref(I(m)))
    return np.array(Af)


def drot(x, y, c, s):
    x = np.ascontiguousarray(x, dtype=np.float64).copy()
    y = np.ascontiguousarray(y, dtype=np.float64).copy()
    _lib.scipy_drot_64_(C.byref(I(len(x))), _p(x), C.byref(I(1)), _p(y), C.byref(I(1)), C.byref(D(c)),
                        C.byref(D(s)))
    return x, y


def dgebrd(A):
    Af = np.asfortranarray(A, dtype=np.float64).copy(order="F")
    m, n = Af.shape
    k = min(m, n)
    d, e, tq, tp = np.zeros(k), np.zeros(max(k - 1, 1)), np.zeros(k), np.zeros(k)
    work = np.zeros(256)
    info = I(0)
    _lib.scipy_dgebrd_64_(C.byref(I(m)), C.byref(I(n)), _p(Af), C.byref(I(m)), _p(d), _p(e), _p(tq), _p(tp),
                          _p(work), C.byref(I(256)), C.byref(info))
    return Af, d, e, tq, tp


def dbdsqr_vt(d, e, ncvt=3):
    d = np.array(d, dtype=np.float64)
    e = np.array(e, dtype=np.float64)
    n = len(d)
    VT = np.asfortranarray(np.eye(n))
    work = np.zeros(4 * n + 16)
    info = I(0)
    dummy = np.zeros(1)
    _lib.scipy_dbdsqr_64_(C.c_char_p(b"U"), C.byref(I(n)), C.byref(I(ncvt)), C.byref(I(0)), C.byref(I(0)),
                          _p(d), _p(e), _p(VT), C.byref(I(n)), _p(dummy), C.byref(I(1)), _p(dummy), C.byref(I(1)),
                          _p(work), C.byref(info), I(1))
    return d, np.array(VT)


def dbdsdc_vt(d, e):
    d = np.array(d, dtype=np.float64)
    e = np.array(e, dtype=np.float64)
    n = len(d)
    U = np.asfortranarray(np.zeros((n, n)))
    VT = np.asfortranarray(np.zeros((n, n)))
    work = np.zeros(3 * n * n + 4 * n + 64)
    iwork = np.zeros(8 * n + 8, dtype=np.int64)
    info = I(0)
    dummy = np.zeros(1)
    _lib.scipy_dbdsdc_64_(C.c_char_p(b"U"), C.c_char_p(b"I"), C.byref(I(n)), _p(d), _p(e), _p(U), C.byref(I(n)),
                          _p(VT), C.byref(I(n)), _p(dummy), _p(dummy), _p(work), _p(iwork), C.byref(info), I(1), I(1))
    return d, np.array(VT)


def dlasdq_vt(d, e):
    d = np.array(d, dtype=np.float64)
    e = np.array(e, dtype=np.float64)
    n = len(d)
    U = np.asfortranarray(np.eye(n))
    VT = np.asfortranarray(np.eye(n))
    work = np.zeros(4 * n + 16)
    info = I(0)
    dummy = np.zeros(1)
    _lib.scipy_dlasdq_64_(C.c_char_p(b"U"), C.byref(I(0)), C.byref(I(n)), C.byref(I(n)), C.byref(I(n)),
                          C.byref(I(0)), _p(d), _p(e), _p(VT), C.byref(I(n)), _p(U), C.byref(I(n)), _p(dummy),
                          C.byref(I(1)), _p(work), C.byref(info), I(1))
    return d, np.array(VT)
