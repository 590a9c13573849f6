"""ctypes wrapper of the plain C schoolbook oracle (oracle/schoolbook.c).
TEST INFRASTRUCTURE ONLY: imported by tests/, smoke() and bench.py's CPU legs.

The same pipeline as ``oracle.hashes`` (Eq. 2, Eq. 4, fold PAPER.md:130-132) but with
schoolbook 32-bit-limb multiplication in C + OpenMP, so larger sizes finish and the CPU
baseline has something honest to time.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "schoolbook.c")
_LIB = os.path.join(_HERE, "_schoolbook.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _LIB, _SRC])
    return _LIB


def _get():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        u64, vp, i32 = ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int
        lib.oracle_mmh.argtypes = [vp, u64, u64, u64, vp, u64, u64, vp, i32]
        lib.oracle_mmh.restype = i32
        lib.oracle_merge.argtypes = [vp, u64, u64, vp]
        lib.oracle_merge.restype = i32
        lib.oracle_mh.argtypes = [vp, u64, vp, vp, u64, u64, vp, i32]
        lib.oracle_mh.restype = i32
        lib.oracle_num_threads.restype = i32
        _lib = lib
    return _lib


def _words(v: int, bits: int) -> np.ndarray:
    nw = (bits + 31) // 32
    return np.frombuffer(v.to_bytes(4 * nw, "little"), dtype="<u4").copy()


def _int(w: np.ndarray) -> int:
    return int.from_bytes(np.ascontiguousarray(w, dtype="<u4").tobytes(), "little")


def num_threads() -> int:
    return int(_get().oracle_num_threads())


def mmh_partial(key, n: int, r: int, gamma: int, a_list, b0: int, b1: int,
                nthreads: int = 0) -> int:
    """sum_{i in [b0,b1)} a_i x_i mod p; a_list[j] = a_{b0+j}."""
    lib = _get()
    key = np.ascontiguousarray(np.asarray(key, dtype=np.uint8))
    wg = (gamma + 31) // 32
    aw = np.concatenate([_words(a, gamma) for a in a_list]) if a_list else np.zeros(0, "<u4")
    y = np.zeros(wg, dtype="<u4")
    rc = lib.oracle_mmh(key.ctypes.data, n, r, gamma, aw.ctypes.data, b0, b1, y.ctypes.data, nthreads)
    if rc != 0:
        raise ValueError(f"oracle_mmh rc={rc}")
    return _int(y)


def merge(ys, gamma: int) -> int:
    lib = _get()
    wg = (gamma + 31) // 32
    parts = np.concatenate([_words(v, gamma) for v in ys])
    y = np.zeros(wg, dtype="<u4")
    lib.oracle_merge(parts.ctypes.data, len(ys), gamma, y.ctypes.data)
    return _int(y)


def mh_output(y: int, gamma: int, b: int, c: int, alpha: int, m: int, nthreads: int = 0) -> bytes:
    lib = _get()
    yw, bw, cw = _words(y, gamma), _words(b, alpha), _words(c, alpha)
    out = np.zeros((m + 7) // 8, dtype=np.uint8)
    rc = lib.oracle_mh(yw.ctypes.data, gamma, bw.ctypes.data, cw.ctypes.data, alpha, m,
                       out.ctypes.data, nthreads)
    if rc != 0:
        raise ValueError(f"oracle_mh rc={rc}")
    return out.tobytes()


def pa_hash(key, n: int, r: int, m: int, gamma: int, a, b: int, c: int, nthreads: int = 0) -> bytes:
    alpha = max(gamma, m)
    k = -(-n // r)
    y = mmh_partial(key, n, r, gamma, list(a), 0, k, nthreads)
    return mh_output(y, gamma, b, c, alpha, m, nthreads)
