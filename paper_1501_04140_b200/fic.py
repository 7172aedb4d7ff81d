"""Thin Python binding of libfic.so (include/fic.h) -- argument marshalling only.

Every step of the encoder runs in the library's CUDA kernels; this module only converts torch
device tensors / numpy arrays to pointers and sizes and checks status codes.  There is no CPU
fallback: if libfic.so is missing or no CUDA device is present, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.environ.get("FIC_SO") or os.path.join(_HERE, "libfic.so")  # (FIC_SO: A/B builds)

RECORD_DTYPE = np.dtype([
    ("rx", "<i4"), ("ry", "<i4"), ("B", "<i4"), ("dom", "<i4"), ("dx", "<i4"), ("dy", "<i4"),
    ("iso", "u1"), ("s_idx", "u1"), ("o_code", "u1"), ("accepted", "u1"), ("err", "<f8"),
], align=True)
RECORD_BYTES = 40
assert RECORD_DTYPE.itemsize == RECORD_BYTES

STATUS = {0: "FIC_OK", 1: "FIC_ERR_ARG", 2: "FIC_ERR_SHAPE", 3: "FIC_ERR_EMPTY_POOL",
          4: "FIC_ERR_CAPACITY", 5: "FIC_ERR_CUDA", 6: "FIC_ERR_NCCL", 7: "FIC_ERR_NOMEM"}

# names exported by include/fic.h (checked by tests/test_abi.py)
EXPORTS = (
    "fic_ctx_create", "fic_ctx_set_stream", "fic_ctx_destroy", "fic_last_error",
    "fic_ctx_set_timing", "fic_get_stats", "fic_build_domain_pool", "fic_pool_info",
    "fic_pool_destroy", "fic_encode_level", "fic_encode", "fic_encode_host", "fic_merge_shards",
    "fic_entropy_lut", "fic_version", "fic_decode", "fic_psnr", "fic_build_domain_pool_topk",
    "fic_encode_topk", "fic_nccl_unique_id", "fic_ctx_create_nccl", "fic_encode_nccl", "fic_encode_nccl_topk",
    "fic_serialize",
)

S_MODE_CODES = {"predefined": 0, "sampled10": 1, "closed5": 2, "grid": 3}  # FIC1 header s_mode


class FicError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class LevelStats(C.Structure):
    _fields_ = [("B", C.c_int32), ("n_candidates", C.c_int64), ("n_kept", C.c_int64),
                ("n_ranges", C.c_int64), ("n_accepted", C.c_int64), ("pairs", C.c_int64),
                ("exact_evals", C.c_int64), ("ms_pool", C.c_float), ("ms_search", C.c_float),
                ("ms_finalize", C.c_float), ("kernel_launches", C.c_int64), ("pairs_scanned", C.c_int64)]


_lib = None


def load(path: str = SO_PATH):
    """Load libfic.so (build it first with paper_1501_04140_b200.build.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built: run python -m paper_1501_04140_b200.build")
    # torch first: its CUDA libraries and NCCL are then the ones libfic.so binds to (one copy
    # of each in the process, whatever the caller imports later)
    import torch  # noqa: F401
    L = C.CDLL(path)
    P, i32, i64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    sig = {
        "fic_ctx_create": ([i32, P, P], C.c_int),
        "fic_ctx_set_stream": ([P, P], C.c_int),
        "fic_ctx_destroy": ([P], C.c_int),
        "fic_last_error": ([P], C.c_char_p),
        "fic_ctx_set_timing": ([P, i32], C.c_int),
        "fic_get_stats": ([P, P, i32, P], C.c_int),
        "fic_build_domain_pool": ([P, P, i32, i32, i32, dbl, P], C.c_int),
        "fic_pool_info": ([P, P, P, P, P, P], C.c_int),
        "fic_pool_destroy": ([P], C.c_int),
        "fic_encode_level": ([P, P, i32, P, P, i64, P, i32, dbl, i32, P], C.c_int),
        "fic_encode": ([P, P, i32, i32, i32, i32, P, P, P, P, i32, i32, P, i64, P], C.c_int),
        "fic_encode_host": ([P, P, i32, i32, i32, i32, P, P, P, P, i32, i32, P, i64, P], C.c_int),
        "fic_merge_shards": ([P, P, P, i32, i64, P], C.c_int),
        "fic_entropy_lut": ([P, i32], C.c_int),
        "fic_decode": ([P, P, i64, i32, i32, i32, P, P, i32, P, P], C.c_int),
        "fic_build_domain_pool_topk": ([P, P, i32, i32, i32, i64, P], C.c_int),
        "fic_encode_topk": ([P, P, i32, i32, i32, i32, P, P, P, P, i32, i32, P, i64, P], C.c_int),
        "fic_nccl_unique_id": ([P], C.c_int),
        "fic_ctx_create_nccl": ([i32, P, P, i32, i32, P], C.c_int),
        "fic_encode_nccl": ([P, P, i32, i32, i32, i32, P, P, P, P, P, i64, P], C.c_int),
        "fic_encode_nccl_topk": ([P, P, i32, i32, i32, i32, P, P, P, P, P, i64, P], C.c_int),
        "fic_psnr": ([P, P, P, i64, P], C.c_int),
        "fic_serialize": ([P, P, i64, i32, i32, i32, i32, P, i32, dbl, P, i64, P], C.c_int),
        "fic_version": ([], C.c_char_p),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _dptr(t) -> C.c_void_p:
    """Device pointer of a contiguous CUDA torch tensor."""
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return C.c_void_p(t.data_ptr())


class _DevArray:
    """__cuda_array_interface__ view of library-owned device memory (zero-copy into torch)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3, "strides": None}


def entropy_lut(mmax: int) -> np.ndarray:
    out = np.zeros(mmax + 1, np.int64)
    st = load().fic_entropy_lut(_ptr(out), mmax)
    if st:
        raise FicError(st, "fic_entropy_lut")
    return out


def version() -> str:
    return load().fic_version().decode()


class Pool:
    """One level's domain pool (library-owned device memory)."""

    def __init__(self, ctx: "Context", handle: C.c_void_p, B: int, L: int, N: int):
        self.ctx, self.handle, self.B, self.L, self.N = ctx, handle, B, L, N

    def info(self):
        import torch
        nc, nk = C.c_int64(), C.c_int64()
        keep, kept, keys = C.c_void_p(), C.c_void_p(), C.c_void_p()
        st = load().fic_pool_info(self.handle, C.byref(nc), C.byref(nk), C.byref(keep),
                                  C.byref(kept), C.byref(keys))
        if st:
            raise FicError(st, "fic_pool_info")
        dev = torch.device("cuda", self.ctx.device)
        out = {"n_candidates": nc.value, "n_kept": nk.value}
        out["keep"] = torch.as_tensor(_DevArray(keep.value, (nc.value,), "|u1"), device=dev).clone()
        out["keys"] = torch.as_tensor(_DevArray(keys.value, (nc.value,), "<i8"), device=dev).clone()
        out["kept"] = (torch.as_tensor(_DevArray(kept.value, (nk.value,), "<i4"), device=dev).clone()
                       if nk.value else torch.zeros(0, dtype=torch.int32, device=dev))
        return out

    def close(self):
        if self.handle:
            load().fic_pool_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Context:
    """A libfic context bound to one CUDA device and the current torch stream."""

    def __init__(self, device: int = 0, stream=None, timing: bool = False, nccl=None):
        """nccl = (unique_id bytes, nranks, rank): also create the context's NCCL communicator
        (fic_ctx_create_nccl; the id from nccl_unique_id() on one rank, shared with all)."""
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("libfic needs a CUDA device (no CPU fallback)")
        self.device = device
        self.lib = load()
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.stream = stream
        h = C.c_void_p()
        if nccl is None:
            st = self.lib.fic_ctx_create(device, C.c_void_p(stream.cuda_stream), C.byref(h))
        else:
            uid, nranks, rank = nccl
            buf = (C.c_uint8 * 128).from_buffer_copy(bytes(uid))
            st = self.lib.fic_ctx_create_nccl(device, C.c_void_p(stream.cuda_stream), buf, int(nranks),
                                              int(rank), C.byref(h))
        if st:
            raise FicError(st, "fic_ctx_create" if nccl is None else "fic_ctx_create_nccl")
        self.handle = h
        self.set_timing(timing)

    # -- plumbing
    def _check(self, st: int, what: str):
        if st != 0:
            msg = self.lib.fic_last_error(self.handle)
            raise FicError(st, f"{what}: {msg.decode() if msg else ''}")

    def set_stream(self, stream):
        self.stream = stream
        self._check(self.lib.fic_ctx_set_stream(self.handle, C.c_void_p(stream.cuda_stream)),
                    "fic_ctx_set_stream")

    def set_timing(self, on):
        """0/False off, 1/True search times only, 2 also pool and finalize times."""
        self._check(self.lib.fic_ctx_set_timing(self.handle, int(on)), "fic_ctx_set_timing")

    def stats(self):
        arr = (LevelStats * 16)()
        n = C.c_int32()
        self._check(self.lib.fic_get_stats(self.handle, arr, 16, C.byref(n)), "fic_get_stats")
        return [{f: getattr(arr[i], f) for f, _ in LevelStats._fields_} for i in range(n.value)]

    def close(self):
        if getattr(self, "handle", None):
            self.lib.fic_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- API
    def build_domain_pool(self, img, B: int, L: int, tau: float = -1.0, topk: int | None = None) -> Pool:
        """Entropy-threshold pool (keep iff H > tau), or the K highest-entropy blocks (topk)."""
        h = C.c_void_p()
        if topk is not None:
            st = self.lib.fic_build_domain_pool_topk(self.handle, _dptr(img), img.shape[0], B, L,
                                                     int(topk), C.byref(h))
        else:
            st = self.lib.fic_build_domain_pool(self.handle, _dptr(img), img.shape[0], B, L,
                                                float(tau), C.byref(h))
        pool = Pool(self, h, B, L, img.shape[0]) if h.value else None
        self._check(st, "fic_build_domain_pool")  # FIC_ERR_EMPTY_POOL raises; pool is freed by GC
        return pool

    def encode_level(self, img, pool: Pool, ranges, s: Sequence[float], rms_tol: float,
                     is_min: bool):
        """ranges: CUDA int32 [n_r, 2] (rx, ry) -> CUDA uint8 [n_r, 40] records (async)."""
        import torch
        n_r = ranges.shape[0]
        out = torch.empty((max(n_r, 1), RECORD_BYTES), dtype=torch.uint8, device=img.device)
        sv = np.ascontiguousarray(s, dtype=np.float64)
        self._check(self.lib.fic_encode_level(self.handle, _dptr(img), img.shape[0], pool.handle,
                                              _dptr(ranges) if n_r else None, n_r, _ptr(sv),
                                              sv.size, float(rms_tol), int(is_min), _dptr(out)),
                    "fic_encode_level")
        return out[:n_r]

    @staticmethod
    def _cfg_arrays(tau, s_sets, rms_tol):
        tau = np.ascontiguousarray(tau, dtype=np.float64)
        n_s = np.array([len(x) for x in s_sets], np.int32)
        s_flat = np.ascontiguousarray(np.concatenate([np.asarray(x, np.float64) for x in s_sets]))
        tol = np.ascontiguousarray(rms_tol, dtype=np.float64)
        return tau, n_s, s_flat, tol

    def encode(self, img, B_max: int, B_min: int, L: int, tau, s_sets, rms_tol, shard: int = 0,
               n_shards: int = 1, out=None, topk=None):
        """Full quadtree encode of a CUDA uint8 [N, N] image -> CUDA uint8 [n, 40] records.
        topk: per-level pool sizes (fic_encode_topk) instead of the entropy thresholds tau."""
        import torch
        N = img.shape[0]
        tau, n_s, s_flat, tol = self._cfg_arrays(tau, s_sets, rms_tol)
        cap = (N // B_min) ** 2
        if out is None or out.shape[0] < cap:
            out = torch.empty((cap, RECORD_BYTES), dtype=torch.uint8, device=img.device)
        n_out = C.c_int64()
        if topk is not None:
            K = np.ascontiguousarray(topk, dtype=np.int64)
            self._check(self.lib.fic_encode_topk(self.handle, _dptr(img), N, B_max, B_min, L, _ptr(K),
                                                 _ptr(s_flat), _ptr(n_s), _ptr(tol), shard, n_shards,
                                                 _dptr(out), out.shape[0], C.byref(n_out)), "fic_encode_topk")
        else:
            self._check(self.lib.fic_encode(self.handle, _dptr(img), N, B_max, B_min, L, _ptr(tau),
                                            _ptr(s_flat), _ptr(n_s), _ptr(tol), shard, n_shards,
                                            _dptr(out), out.shape[0], C.byref(n_out)), "fic_encode")
        return out[: n_out.value]

    def encode_host(self, img: np.ndarray, B_max: int, B_min: int, L: int, tau, s_sets, rms_tol,
                    shard: int = 0, n_shards: int = 1, out: np.ndarray | None = None):
        """Same through host buffers (H2D of the image and D2H of the records inside the call)."""
        img = np.ascontiguousarray(img, dtype=np.uint8)
        N = img.shape[0]
        tau, n_s, s_flat, tol = self._cfg_arrays(tau, s_sets, rms_tol)
        cap = (N // B_min) ** 2
        if out is None or out.shape[0] < cap:
            out = np.zeros(cap, RECORD_DTYPE)
        n_out = C.c_int64()
        self._check(self.lib.fic_encode_host(self.handle, _ptr(img), N, B_max, B_min, L,
                                             _ptr(tau), _ptr(s_flat), _ptr(n_s), _ptr(tol), shard,
                                             n_shards, _ptr(out), out.shape[0], C.byref(n_out)),
                    "fic_encode_host")
        return out[: n_out.value]

    def encode_cfg(self, cfg, img, **kw):
        kw.setdefault("topk", cfg.get("topk"))
        return self.encode(img, cfg["B_max"], cfg["B_min"], cfg["L"], cfg["tau"], cfg["s"],
                           cfg["rms_tol"], **kw)

    def merge_shards(self, recs, counts: Sequence[int], stride: int):
        """recs: CUDA uint8 [n_shards * stride, 40] -> CUDA uint8 [sum(counts), 40]."""
        import torch
        cnt = np.ascontiguousarray(counts, dtype=np.int64)
        out = torch.empty((max(int(cnt.sum()), 1), RECORD_BYTES), dtype=torch.uint8,
                          device=recs.device)
        self._check(self.lib.fic_merge_shards(self.handle, _dptr(recs), _ptr(cnt), cnt.size,
                                              stride, _dptr(out)), "fic_merge_shards")
        return out[: int(cnt.sum())]

    def encode_nccl(self, img, B_max: int, B_min: int, L: int, tau, s_sets, rms_tol, out=None, topk=None):
        """Sharded encode over the context's NCCL communicator (fic_encode_nccl, or
        fic_encode_nccl_topk with per-level pool sizes): every rank gets the full canonical code
        (CUDA uint8 [n, 40])."""
        import torch
        N = img.shape[0]
        tau, n_s, s_flat, tol = self._cfg_arrays(tau, s_sets, rms_tol)
        cap = (N // B_min) ** 2
        if out is None or out.shape[0] < cap:
            out = torch.empty((cap, RECORD_BYTES), dtype=torch.uint8, device=img.device)
        n_out = C.c_int64()
        if topk is None:
            st = self.lib.fic_encode_nccl(self.handle, _dptr(img), N, B_max, B_min, L, _ptr(tau), _ptr(s_flat),
                                          _ptr(n_s), _ptr(tol), _dptr(out), out.shape[0], C.byref(n_out))
            self._check(st, "fic_encode_nccl")
        else:
            K = np.ascontiguousarray(topk, dtype=np.int64)
            st = self.lib.fic_encode_nccl_topk(self.handle, _dptr(img), N, B_max, B_min, L, _ptr(K), _ptr(s_flat),
                                               _ptr(n_s), _ptr(tol), _dptr(out), out.shape[0], C.byref(n_out))
            self._check(st, "fic_encode_nccl_topk")
        return out[: n_out.value]

    def encode_nccl_cfg(self, cfg, img, out=None):
        return self.encode_nccl(img, cfg["B_max"], cfg["B_min"], cfg["L"], cfg["tau"], cfg["s"], cfg["rms_tol"],
                                out=out, topk=cfg.get("topk"))

    def decode(self, recs, N: int, B_max: int, s_sets, iterations: int = 12, init=None):
        """PIFS decode (fic_decode): CUDA uint8 [n, 40] records -> CUDA uint8 [N, N] image."""
        import torch
        n_s = np.array([len(x) for x in s_sets], np.int32)
        s_flat = np.ascontiguousarray(np.concatenate([np.asarray(x, np.float64) for x in s_sets]))
        dev = recs.device if recs.is_cuda else torch.device("cuda")
        out = torch.empty((N, N), dtype=torch.uint8, device=dev)
        n = recs.shape[0]
        self._check(self.lib.fic_decode(self.handle, _dptr(recs) if n else None, n, N, B_max, len(s_sets),
                                        _ptr(s_flat), _ptr(n_s), int(iterations),
                                        _dptr(init) if init is not None else None, _dptr(out)),
                    "fic_decode")
        return out

    def serialize(self, recs, N: int, B_max: int, B_min: int, L: int, s_sets, s_mode: str = "predefined",
                  s_max: float = 1.0) -> bytes:
        """FIC1 stream of a code (fic_serialize): recs = CUDA uint8 [n, 40] records (one per leaf)."""
        import torch
        n_s = np.ascontiguousarray([len(s) for s in s_sets], dtype=np.int32)
        n = recs.shape[0]
        cap = 64 + len(s_sets) + n * 8
        out = torch.empty(cap, dtype=torch.uint8, device=recs.device)
        nb = C.c_int64()
        self._check(self.lib.fic_serialize(self.handle, _dptr(recs), n, N, B_max, B_min, L, _ptr(n_s),
                                           S_MODE_CODES[s_mode], float(s_max), _dptr(out), cap, C.byref(nb)),
                    "fic_serialize")
        return bytes(out[: nb.value].cpu().numpy().tobytes())

    def serialize_cfg(self, cfg, recs) -> bytes:
        return self.serialize(recs, cfg["N"], cfg["B_max"], cfg["B_min"], cfg["L"], cfg["s"],
                              cfg.get("s_mode", "predefined"))

    def psnr(self, a, b) -> float:
        """PSNR of two CUDA uint8 images (fic_psnr)."""
        v = C.c_double()
        self._check(self.lib.fic_psnr(self.handle, _dptr(a), _dptr(b), a.numel(), C.byref(v)), "fic_psnr")
        return v.value


def nccl_unique_id() -> bytes:
    """A fresh NCCL unique id (128 bytes) for Context(nccl=(id, nranks, rank))."""
    buf = (C.c_uint8 * 128)()
    st = load().fic_nccl_unique_id(buf)
    if st:
        raise FicError(st, "fic_nccl_unique_id")
    return bytes(buf)


def records_to_numpy(t) -> np.ndarray:
    """CUDA/CPU uint8 [n, 40] tensor -> numpy structured array (RECORD_DTYPE)."""
    a = t.detach().cpu().contiguous().numpy()
    return a.reshape(-1).view(RECORD_DTYPE).copy() if a.size else np.zeros(0, RECORD_DTYPE)
