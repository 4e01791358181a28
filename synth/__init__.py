"""Seeded synthetic inputs shared by the oracle and the CUDA path.

Holds none of the method's arithmetic: only graph / opinion generators
(counter-based, so results do not depend on thread count).  See synth.c for
the recipes and DESIGN.md "Input recipe" for how they stand in for the paper's
datasets (§5).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libsynth.so")
_lib = None

MASK64 = (1 << 64) - 1
STREAM_OPINION = 0x1
STREAM_WEIGHT = 0x5 << 40


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "synth.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _SO, src, "-lm"])
    return _SO


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        i64, u64, dbl, ptr = ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p
        lib.synth_rand64.restype = u64
        lib.synth_rand64.argtypes = [u64, u64, u64]
        lib.synth_opinions.restype = ctypes.c_int
        lib.synth_opinions.argtypes = [ctypes.c_int, u64, i64, ptr]
        lib.synth_er.restype = i64
        lib.synth_er.argtypes = [i64, dbl, u64, ptr, ptr, i64]
        lib.synth_ba.restype = i64
        lib.synth_ba.argtypes = [i64, i64, u64, ptr, ptr, i64]
        lib.synth_rmat.restype = i64
        lib.synth_rmat.argtypes = [ctypes.c_int, i64, dbl, dbl, dbl, u64, ptr, ptr, i64]
        lib.synth_weights_u8.restype = ctypes.c_int
        lib.synth_weights_u8.argtypes = [u64, i64, ptr, ptr, ptr]
        lib.synth_num_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# ---------------------------------------------------------------- numpy mirror of rand64
def _sm64(x: np.ndarray) -> np.ndarray:
    x = (x + np.uint64(0x9E3779B97F4A7C15)) & np.uint64(MASK64)
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def rand64_np(seed: int, stream: int, ctr: np.ndarray) -> np.ndarray:
    """numpy mirror of synth_rand64 (used to cross-check the C generator)."""
    with np.errstate(over="ignore"):
        k = _sm64(np.array([seed], dtype=np.uint64)) ^ np.uint64(stream)
        k = _sm64(k)
        return _sm64(k ^ np.asarray(ctr, dtype=np.uint64))


def rand64(seed: int, stream: int, ctr: int) -> int:
    return int(_L().synth_rand64(seed, stream, ctr))


# ---------------------------------------------------------------- generators
OPINION_KINDS = {"uniform": 0, "exponential": 1, "powerlaw": 2}


def opinions(kind: str, n: int, seed: int) -> np.ndarray:
    s = np.empty(n, dtype=np.float64)
    rc = _L().synth_opinions(OPINION_KINDS[kind], seed, n, _p(s))
    if rc != 0:
        raise ValueError("synth_opinions failed")
    return s


def erdos_renyi(n: int, p: float, seed: int):
    L = _L()
    m = L.synth_er(n, p, seed, None, None, 0)
    if m < 0:
        raise ValueError("bad ER parameters")
    u = np.empty(m, dtype=np.int32)
    v = np.empty(m, dtype=np.int32)
    m2 = L.synth_er(n, p, seed, _p(u), _p(v), m)
    assert m2 == m
    return u, v


def barabasi_albert(n: int, m: int, seed: int):
    L = _L()
    tot = L.synth_ba(n, m, seed, None, None, 0)
    if tot < 0:
        raise ValueError("bad BA parameters")
    u = np.empty(tot, dtype=np.int32)
    v = np.empty(tot, dtype=np.int32)
    got = L.synth_ba(n, m, seed, _p(u), _p(v), tot)
    assert got == tot
    return u, v


def rmat(scale: int, edge_factor: int, a: float, b: float, c: float, seed: int):
    L = _L()
    m = L.synth_rmat(scale, edge_factor, a, b, c, seed, None, None, 0)
    if m < 0:
        raise ValueError("bad R-MAT parameters")
    u = np.empty(m, dtype=np.int32)
    v = np.empty(m, dtype=np.int32)
    got = L.synth_rmat(scale, edge_factor, a, b, c, seed, _p(u), _p(v), m)
    assert got == m
    return u, v


def weights_u8(u: np.ndarray, v: np.ndarray, seed: int) -> np.ndarray:
    w = np.empty(len(u), dtype=np.uint8)
    _L().synth_weights_u8(seed, len(u), _p(np.ascontiguousarray(u)), _p(np.ascontiguousarray(v)), _p(w))
    return w


def num_threads() -> int:
    return int(_L().synth_num_threads())


from .configs import CONFIGS, make_config  # noqa: E402,F401
