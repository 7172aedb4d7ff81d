"""ctypes wrapper around oracle/fic_oracle.c (TEST INFRASTRUCTURE ONLY; see __init__.py)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fic_oracle.c")
_SO = os.path.join(_HERE, "libfic_oracle.so")
_lock = threading.Lock()
_lib = None

RECORD_DTYPE = np.dtype([
    ("rx", "<i4"), ("ry", "<i4"), ("B", "<i4"), ("dom", "<i4"), ("dx", "<i4"), ("dy", "<i4"),
    ("iso", "u1"), ("s_idx", "u1"), ("o_code", "u1"), ("accepted", "u1"), ("err", "<f8"),
], align=True)
assert RECORD_DTYPE.itemsize == 40


def build(force: bool = False) -> str:
    """Compile the oracle with gcc: -O2, no FMA contraction, no fast-math, OpenMP."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-fPIC", "-shared", "-o", _SO + ".tmp", _SRC, "-lquadmath", "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(_SO + ".tmp", _SO)
    return _SO


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_SO)
            P = C.c_void_p
            L.fico_lut.argtypes = [P, C.c_int32]
            L.fico_threshold.argtypes = [C.c_double, C.c_int32]
            L.fico_threshold.restype = C.c_int64
            L.fico_axis_candidates.argtypes = [C.c_int32] * 3
            L.fico_axis_candidates.restype = C.c_int64
            L.fico_entropy_keys.argtypes = [P, C.c_int32, C.c_int32, C.c_int32, C.c_double, P, P, P]
            L.fico_kept_list.argtypes = [P, C.c_int32, C.c_int32, C.c_int32, C.c_double, P]
            L.fico_kept_list.restype = C.c_int64
            L.fico_apply_isometry.argtypes = [P, C.c_int32, C.c_int32, P]
            L.fico_decimate.argtypes = [P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, P]
            L.fico_o_code.argtypes = [C.c_double]
            L.fico_o_code.restype = C.c_int32
            L.fico_encode_level.argtypes = [P, C.c_int32, C.c_int32, C.c_int32, P, C.c_int64, P,
                                            C.c_int64, P, C.c_int32, C.c_double, C.c_int32, P]
            L.fico_encode.argtypes = [P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, P, P, P, P,
                                      C.c_int32, C.c_int32, P, C.c_int64, P]
            L.fico_num_threads.restype = C.c_int
            L.fico_kept_list_topk.argtypes = [P, C.c_int32, C.c_int32, C.c_int32, C.c_int64, P]
            L.fico_kept_list_topk.restype = C.c_int64
            L.fico_encode_sel.argtypes = [P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, P, P, P, P, P,
                                          C.c_int32, C.c_int32, P, C.c_int64, P]
            L.fico_o_value.argtypes = [C.c_int32]
            L.fico_o_value.restype = C.c_double
            L.fico_decode.argtypes = [P, C.c_int64, C.c_int32, P, P, C.c_int32, C.c_int32, C.c_int32, P, P]
            L.fico_psnr.argtypes = [P, P, C.c_int64]
            L.fico_psnr.restype = C.c_double
            _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _img(img):
    a = np.ascontiguousarray(img, dtype=np.uint8)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ValueError("square 2-D uint8 image expected")
    return a


def num_threads() -> int:
    return int(lib().fico_num_threads())


def lut(mmax: int) -> np.ndarray:
    out = np.zeros(mmax + 1, dtype=np.int64)
    lib().fico_lut(_p(out), mmax)
    return out


def threshold(tau: float, m: int) -> int:
    return int(lib().fico_threshold(float(tau), int(m)))


def axis_candidates(N: int, B: int, L: int) -> int:
    return int(lib().fico_axis_candidates(N, B, L))


def entropy_keys(img, B: int, L: int, tau: float = -1.0):
    """-> (keys int64 [n_c], keep uint8 [n_c], H float64 [n_c]) in row-major candidate order."""
    a = _img(img)
    A = axis_candidates(a.shape[0], B, L)
    if A <= 0:
        raise ValueError("no candidates")
    keys = np.zeros(A * A, np.int64)
    keep = np.zeros(A * A, np.uint8)
    H = np.zeros(A * A, np.float64)
    st = lib().fico_entropy_keys(_p(a), a.shape[0], B, L, float(tau), _p(keys), _p(keep), _p(H))
    if st:
        raise RuntimeError(f"fico_entropy_keys status {st}")
    return keys, keep, H


def kept_list(img, B: int, L: int, tau: float) -> np.ndarray:
    a = _img(img)
    A = axis_candidates(a.shape[0], B, L)
    out = np.zeros(max(A * A, 1), np.int32)
    n = lib().fico_kept_list(_p(a), a.shape[0], B, L, float(tau), _p(out))
    if n < 0:
        raise RuntimeError(f"fico_kept_list status {-n}")
    return out[:n].copy()


def kept_list_topk(img, B: int, L: int, K: int) -> np.ndarray:
    """Top-K selection (reading R27): K largest entropy keys, ties to the lower index; row-major."""
    a = _img(img)
    A = axis_candidates(a.shape[0], B, L)
    out = np.zeros(max(A * A, 1), np.int32)
    n = lib().fico_kept_list_topk(_p(a), a.shape[0], B, L, int(K), _p(out))
    if n < 0:
        raise RuntimeError(f"fico_kept_list_topk status {-n}")
    return out[:n].copy()


def isometry(X: np.ndarray, k: int) -> np.ndarray:
    X = np.ascontiguousarray(X, dtype=np.int32)
    out = np.zeros_like(X)
    lib().fico_apply_isometry(_p(X), X.shape[0], int(k), _p(out))
    return out


def decimate(img, x: int, y: int, B: int) -> np.ndarray:
    a = _img(img)
    out = np.zeros((B, B), np.int32)
    lib().fico_decimate(_p(a), a.shape[0], x, y, B, _p(out))
    return out


def o_code(o: float) -> int:
    return int(lib().fico_o_code(float(o)))


def encode_level(img, B: int, L: int, kept, ranges, s, rms_tol: float, is_min: bool):
    """Records (RECORD_DTYPE) for each range of `ranges` ([n_r, 2] int32 (rx, ry))."""
    a = _img(img)
    kept = np.ascontiguousarray(kept, dtype=np.int32)
    ranges = np.ascontiguousarray(np.asarray(ranges, dtype=np.int32).reshape(-1, 2))
    s = np.ascontiguousarray(s, dtype=np.float64)
    out = np.zeros(ranges.shape[0], RECORD_DTYPE)
    st = lib().fico_encode_level(_p(a), a.shape[0], B, L, _p(kept), kept.size, _p(ranges),
                                 ranges.shape[0], _p(s), s.size, float(rms_tol), int(is_min),
                                 _p(out))
    if st:
        raise RuntimeError(f"fico_encode_level status {st}")
    return out


def encode(img, B_max, B_min, L, tau, s_sets, rms_tol, shard=0, n_shards=1, topk=None):
    """Full quadtree encode -> records of accepted leaves (B desc, then (ry, rx)).
    topk: per-level pool sizes (reading R27) instead of the entropy thresholds tau."""
    a = _img(img)
    tau = np.ascontiguousarray(tau, dtype=np.float64)
    tk = None if topk is None else np.ascontiguousarray(topk, dtype=np.int64)
    n_s = np.array([len(x) for x in s_sets], np.int32)
    s_flat = np.ascontiguousarray(np.concatenate([np.asarray(x, np.float64) for x in s_sets]))
    tol = np.ascontiguousarray(rms_tol, dtype=np.float64)
    N = a.shape[0]
    cap = max(1, (N // B_min) ** 2)
    out = np.zeros(cap, RECORD_DTYPE)
    n_out = np.zeros(1, np.int64)
    st = lib().fico_encode_sel(_p(a), N, B_max, B_min, L, _p(tau), None if tk is None else _p(tk),
                               _p(s_flat), _p(n_s), _p(tol), shard, n_shards, _p(out), cap, _p(n_out))
    if st:
        raise RuntimeError(f"fico_encode status {st}")
    return out[: int(n_out[0])].copy()


def encode_cfg(cfg, img=None, shard=0, n_shards=1):
    from fic_inputs import image_for
    if img is None:
        img = image_for(cfg)
    return encode(img, cfg["B_max"], cfg["B_min"], cfg["L"], cfg["tau"], cfg["s"],
                  cfg["rms_tol"], shard, n_shards, cfg.get("topk"))


def o_value(code: int) -> float:
    """Dequantised offset of an o code (centre of the [R11] cell), reading R23."""
    return float(lib().fico_o_value(int(code)))


def decode(records, N: int, s_sets, B_max: int, iterations: int = 12, init=None):
    """PIFS decode (readings R23-R26): Jacobi iterations from the constant 128 image (or init)."""
    rec = np.ascontiguousarray(records, dtype=RECORD_DTYPE)
    n_s = np.array([len(x) for x in s_sets], np.int32)
    s_flat = np.ascontiguousarray(np.concatenate([np.asarray(x, np.float64) for x in s_sets]))
    out = np.zeros((N, N), np.uint8)
    ini = None if init is None else _img(init)
    st = lib().fico_decode(_p(rec), rec.shape[0], N, _p(s_flat), _p(n_s), B_max, len(s_sets), iterations,
                           None if ini is None else _p(ini), _p(out))
    if st:
        raise RuntimeError(f"fico_decode status {st}")
    return out


def psnr(a, b) -> float:
    a = np.ascontiguousarray(a, dtype=np.uint8)
    b = np.ascontiguousarray(b, dtype=np.uint8)
    if a.shape != b.shape:
        raise ValueError("shape mismatch")
    return float(lib().fico_psnr(_p(a), _p(b), a.size))
