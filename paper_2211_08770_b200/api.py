"""Thin Python binding over libtt_b200 (same names as include/tt_b200.h).

Argument marshalling only: every arithmetic step runs in the sm_100a kernels of the
shared library.  torch provides device memory (input cores) and the CUDA stream.
"""
from __future__ import annotations

import ctypes as C
import math
from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import _native as N

DEFAULT_FLOOR_C = 2048.0


class _CoreArray:
    """Zero-copy __cuda_array_interface__ over a library-owned core."""

    def __init__(self, ptr: int, shape, owner):
        self._owner = owner
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f8", "data": (ptr, False),
                                         "version": 3, "strides": None, "stream": None}


class Context:
    def __init__(self, device: int = 0, stream: Optional[torch.cuda.Stream] = None):
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2211_08770_b200 needs a CUDA device (B200, sm_100a); no CPU fallback")
        self.lib = N.load()
        self.device = device
        torch.cuda.set_device(device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        h = C.c_void_p()
        st = self.lib.tt_ctx_create(device, C.c_void_p(self.stream.cuda_stream), C.byref(h))
        if st != 0:
            raise N.TTError(st, "tt_ctx_create failed")
        self.handle = h

    def check(self, st: int):
        if st != 0:
            raise N.TTError(st, self.lib.tt_last_error(self.handle).decode())

    @property
    def launches(self) -> int:
        return int(self.lib.tt_ctx_launch_count(self.handle))

    def profile(self, enable: bool):
        self.check(self.lib.tt_ctx_profile(self.handle, int(enable)))

    def profile_report(self) -> dict:
        """{class: {launches, ms, flops, bytes}} from the event timing of tt_ctx_profile."""
        out = {}
        i = 0
        while True:
            name = C.create_string_buffer(64)
            l, ms, fl, by = C.c_int64(), C.c_double(), C.c_double(), C.c_double()
            st = self.lib.tt_ctx_profile_query(self.handle, i, name, 64, C.byref(l), C.byref(ms), C.byref(fl),
                                               C.byref(by))
            if st != 0:
                break
            out[name.value.decode()] = {"launches": l.value, "ms": ms.value, "flops": fl.value, "bytes": by.value}
            i += 1
        return out

    def sync(self):
        self.check(self.lib.tt_ctx_sync(self.handle))

    def close(self):
        if getattr(self, "handle", None):
            self.lib.tt_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DeviceTT:
    """Caller-owned TT-vector whose cores are torch CUDA float64 tensors (r_{k-1}, n_k, r_k)."""

    def __init__(self, cores: Sequence[torch.Tensor], norm: float = float("nan")):
        self.cores = [c.contiguous() for c in cores]
        for c in self.cores:
            if not (c.is_cuda and c.dtype == torch.float64 and c.dim() == 3):
                raise ValueError("cores must be 3-D float64 CUDA tensors")
        self.norm = float(norm)

    @staticmethod
    def from_numpy(cores: Sequence[np.ndarray], device="cuda", norm: float = float("nan")) -> "DeviceTT":
        return DeviceTT([torch.from_numpy(np.ascontiguousarray(c, dtype=np.float64)).to(device) for c in cores], norm)

    @property
    def d(self):
        return len(self.cores)

    @property
    def ranks(self):
        return [self.cores[0].shape[0]] + [c.shape[2] for c in self.cores]

    @property
    def modes(self):
        return [c.shape[1] for c in self.cores]

    def _view(self):
        d = self.d
        n = (C.c_int64 * d)(*self.modes)
        r = (C.c_int64 * (d + 1))(*self.ranks)
        core = (C.c_void_p * d)(*[c.data_ptr() for c in self.cores])
        v = N.TTView(d, C.cast(n, C.POINTER(C.c_int64)), C.cast(r, C.POINTER(C.c_int64)),
                     C.cast(core, C.POINTER(C.c_void_p)), self.norm)
        return v, (n, r, core, self)

    def to_numpy(self) -> List[np.ndarray]:
        return [c.cpu().numpy() for c in self.cores]


class LibTT:
    """Library-owned TT-vector (result of a rounding / sum); freed with the object."""

    def __init__(self, ctx: Context, handle: C.c_void_p):
        self.ctx = ctx
        self.handle = handle
        v = N.TTView()
        ctx.check(ctx.lib.tt_tensor_view(handle, C.byref(v)))
        self.d = v.d
        self.modes = [v.n[k] for k in range(v.d)]
        self.ranks = [v.r[k] for k in range(v.d + 1)]
        self.norm = v.norm
        self._ptrs = [v.core[k] for k in range(v.d)]

    def _view(self):
        v = N.TTView()
        self.ctx.check(self.ctx.lib.tt_tensor_view(self.handle, C.byref(v)))
        return v, (self,)

    def to_numpy(self) -> List[np.ndarray]:
        shapes = [(self.ranks[k], self.modes[k], self.ranks[k + 1]) for k in range(self.d)]
        outs = [np.empty(s, dtype=np.float64) for s in shapes]
        ptrs = (C.c_void_p * self.d)(*[o.ctypes.data for o in outs])
        self.ctx.check(self.ctx.lib.tt_download(self.ctx.handle, self.handle, ptrs))
        return outs

    def cores_torch(self) -> List[torch.Tensor]:
        """Zero-copy torch views of the cores (valid while this object lives)."""
        out = []
        for k in range(self.d):
            shp = (self.ranks[k], self.modes[k], self.ranks[k + 1])
            out.append(torch.as_tensor(_CoreArray(self._ptrs[k], shp, self), device=f"cuda:{self.ctx.device}"))
        return out

    def free(self):
        if self.handle is not None and self.ctx.handle is not None:
            self.ctx.lib.tt_tensor_free(self.ctx.handle, self.handle)
        self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _views(tts):
    arr = (N.TTView * len(tts))()
    keep = []
    for i, t in enumerate(tts):
        v, k = t._view()
        arr[i] = v
        keep.append(k)
    return arr, keep


def _opts(rel_tol, floor_c, max_rank, theta, rank_revealing=True):
    return N.RoundOpts(float(rel_tol), int(max_rank), float(floor_c), float(theta), int(bool(rank_revealing)))


# ----------------------------------------------------------------------------- entry points
def tt_round(ctx: Context, terms, coeffs, rel_tol: float, floor_c: float = DEFAULT_FLOOR_C,
             max_rank: int = 0, theta: float = 0.5, rank_revealing: bool = True) -> Tuple[LibTT, dict]:
    arr, keep = _views(terms)
    cf = (C.c_double * len(terms))(*[float(c) for c in coeffs])
    o = _opts(rel_tol, floor_c, max_rank, theta, rank_revealing)
    h = C.c_void_p()
    info = N.RoundInfo()
    ctx.check(ctx.lib.tt_round(ctx.handle, len(terms), cf, arr, C.byref(o), C.byref(h), C.byref(info)))
    return LibTT(ctx, h), {"norm": info.norm, "scale": info.scale, "tau": info.tau,
                           "qrcp_steps": info.qrcp_steps, "resumes": info.resumes}


def tt_round_batch(ctx: Context, items, rel_tol: float, floor_c: float = DEFAULT_FLOOR_C, max_rank: int = 0,
                   theta: float = 0.5, rank_revealing: bool = True) -> List[LibTT]:
    B = len(items)
    Ks = (C.c_int32 * B)(*[len(t) for t, _ in items])
    keep = []
    vptrs = (C.POINTER(N.TTView) * B)()
    cptrs = (C.POINTER(C.c_double) * B)()
    for b, (terms, coeffs) in enumerate(items):
        arr, k = _views(terms)
        cf = (C.c_double * len(coeffs))(*[float(c) for c in coeffs])
        keep += [arr, k, cf]
        vptrs[b] = C.cast(arr, C.POINTER(N.TTView))
        cptrs[b] = C.cast(cf, C.POINTER(C.c_double))
    outs = (C.c_void_p * B)()
    o = _opts(rel_tol, floor_c, max_rank, theta, rank_revealing)
    ctx.check(ctx.lib.tt_round_batch(ctx.handle, B, Ks, cptrs, vptrs, C.byref(o), outs, None))
    return [LibTT(ctx, C.c_void_p(outs[b])) for b in range(B)]


class BatchTT:
    """Result of tt_round_batch_strided: B rounded TT-vectors owned by one library handle."""

    def __init__(self, ctx: Context, handle: C.c_void_p):
        self.ctx = ctx
        self.handle = handle
        B, d = C.c_int32(), C.c_int32()
        ctx.check(ctx.lib.tt_batch_shape(handle, C.byref(B), C.byref(d)))
        self.B, self.d = B.value, d.value
        rk = np.empty((self.B, self.d + 1), dtype=np.int64)
        nr = np.empty(self.B, dtype=np.float64)
        if self.B:
            ctx.check(ctx.lib.tt_batch_ranks(handle, rk.ctypes.data_as(C.POINTER(C.c_int64)),
                                             nr.ctypes.data_as(C.POINTER(C.c_double))))
        self.ranks = rk
        self.norms = nr

    def __len__(self):
        return self.B

    def view(self, b: int):
        v = N.TTView()
        self.ctx.check(self.ctx.lib.tt_batch_view(self.handle, int(b), C.byref(v)))
        return v

    def cores_torch(self, b: int) -> List[torch.Tensor]:
        """Zero-copy torch views of item b's cores (valid while this object lives)."""
        v = self.view(b)
        out = []
        for k in range(self.d):
            shp = (int(v.r[k]), int(v.n[k]), int(v.r[k + 1]))
            out.append(torch.as_tensor(_CoreArray(v.core[k], shp, self), device=f"cuda:{self.ctx.device}"))
        return out

    def arenas(self):
        """[(device pointer, doubles)] of the result arenas: items in order, cores in order."""
        out, w = [], 0
        while True:
            ptr, cnt = C.c_void_p(), C.c_int64()
            st = self.ctx.lib.tt_batch_arena(self.handle, w, C.byref(ptr), C.byref(cnt))
            if st == 3:  # TT_EINDEX: past the last arena
                return out
            self.ctx.check(st)
            out.append((int(ptr.value or 0), int(cnt.value)))
            w += 1

    def total_doubles(self) -> int:
        cnt = C.c_int64()
        st = self.ctx.lib.tt_batch_download(self.ctx.handle, self.handle, None, 0, C.byref(cnt))
        if st not in (0, 1):
            self.ctx.check(st)
        return int(cnt.value)

    def download(self, host: torch.Tensor) -> int:
        """Copy every result core into the (pinned) float64 CPU tensor `host`, items in order;
        returns the number of doubles written."""
        cnt = C.c_int64()
        self.ctx.check(self.ctx.lib.tt_batch_download(self.ctx.handle, self.handle, C.c_void_p(host.data_ptr()),
                                                      int(host.numel()), C.byref(cnt)))
        return int(cnt.value)

    def item_numpy(self, b: int) -> List[np.ndarray]:
        return [c.cpu().numpy() for c in self.cores_torch(b)]

    def free(self):
        if self.handle is not None and self.ctx.handle is not None:
            self.ctx.lib.tt_batch_free(self.ctx.handle, self.handle)
        self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def tt_round_batch_strided(ctx: Context, terms, coeffs, rel_tol: float, norms=None,
                           floor_c: float = DEFAULT_FLOOR_C, max_rank: int = 0) -> BatchTT:
    """terms[l][k]: CUDA float64 tensor (B, r_{k-1}, n_k, r_k) holding core k of term l of every
    item (item stride = its first-dimension stride); coeffs, norms: (B, K) array-likes (norms
    optional: computed on the device)."""
    K = len(terms)
    d = len(terms[0])
    B = int(terms[0][0].shape[0])
    n = (C.c_int64 * d)(*[int(terms[0][k].shape[2]) for k in range(d)])
    r = (C.c_int64 * (K * (d + 1)))()
    base = (C.c_void_p * (K * d))()
    stride = (C.c_int64 * (K * d))()
    for l in range(K):
        r[l * (d + 1)] = int(terms[l][0].shape[1])
        for k in range(d):
            t = terms[l][k]
            if not (t.is_cuda and t.dtype == torch.float64 and t.dim() == 4 and t[0].is_contiguous()):
                raise ValueError("terms[l][k] must be (B, r0, n, r1) float64 CUDA tensors with contiguous items")
            if int(t.shape[0]) != B:
                raise ValueError("all term cores need the same batch size B")
            r[l * (d + 1) + k + 1] = int(t.shape[3])
            base[l * d + k] = t.data_ptr()
            stride[l * d + k] = int(t.stride(0)) if B > 1 else 0
    cf = np.ascontiguousarray(np.asarray(coeffs, dtype=np.float64).reshape(B, K))
    nr = None if norms is None else np.ascontiguousarray(np.asarray(norms, dtype=np.float64).reshape(B, K))
    o = _opts(rel_tol, floor_c, max_rank, 0.5, False)
    h = C.c_void_p()
    ctx.check(ctx.lib.tt_round_batch_strided(
        ctx.handle, B, K, d, n, r, base, stride, cf.ctypes.data_as(C.POINTER(C.c_double)),
        None if nr is None else nr.ctypes.data_as(C.POINTER(C.c_double)), C.byref(o), C.byref(h)))
    return BatchTT(ctx, h)


def tt_round_batch_host(ctx: Context, host_terms, coeffs, rel_tol: float, norms=None,
                        floor_c: float = DEFAULT_FLOOR_C, max_rank: int = 0, slices: int = 4,
                        out_host: Optional[torch.Tensor] = None):
    """End-to-end batched rounding from HOST inputs to HOST results: one call of the C ABI's
    tt_round_batch_host (the library pipelines host->device copies, the rounding and the
    device->host copies over `slices` slices on its own streams).
    host_terms[l][k]: CPU float64 tensors (B, r_{k-1}, n_k, r_k), pinned for overlap.  Results go
    to out_host (float64, items in order, cores in order, each core C order); when it is None or
    too small a pinned buffer is allocated (and the call repeated if the first estimate was too
    small).  Returns (out_host, ranks (B, d+1), norms (B,), doubles written)."""
    K, d = len(host_terms), len(host_terms[0])
    B = int(host_terms[0][0].shape[0])
    n = (C.c_int64 * d)(*[int(host_terms[0][k].shape[2]) for k in range(d)])
    r = (C.c_int64 * (K * (d + 1)))()
    base = (C.c_void_p * (K * d))()
    stride = (C.c_int64 * (K * d))()
    in_doubles = 0
    for l in range(K):
        r[l * (d + 1)] = int(host_terms[l][0].shape[1])
        for k in range(d):
            t = host_terms[l][k]
            if not (t.device.type == "cpu" and t.dtype == torch.float64 and t.dim() == 4 and t[0].is_contiguous()):
                raise ValueError("host_terms[l][k] must be (B, r0, n, r1) float64 CPU tensors with contiguous items")
            if int(t.shape[0]) != B:
                raise ValueError("all term cores need the same batch size B")
            r[l * (d + 1) + k + 1] = int(t.shape[3])
            base[l * d + k] = t.data_ptr()
            stride[l * d + k] = int(t.stride(0)) if B > 1 else 0
            in_doubles += int(t[0].numel())
    cf = np.ascontiguousarray(np.asarray(coeffs, dtype=np.float64).reshape(B, K))
    nr = None if norms is None else np.ascontiguousarray(np.asarray(norms, dtype=np.float64).reshape(B, K))
    o = _opts(rel_tol, floor_c, max_rank, 0.5, False)
    ranks = np.empty((B, d + 1), dtype=np.int64)
    nrm = np.empty(B, dtype=np.float64)
    if out_host is None:
        out_host = torch.empty(max(B * in_doubles, 1), dtype=torch.float64).pin_memory()
    for _ in range(2):
        cnt = C.c_int64()
        st = ctx.lib.tt_round_batch_host(
            ctx.handle, B, K, d, n, r, base, stride, cf.ctypes.data_as(C.POINTER(C.c_double)),
            None if nr is None else nr.ctypes.data_as(C.POINTER(C.c_double)), C.byref(o), int(slices),
            C.c_void_p(out_host.data_ptr()), int(out_host.numel()), C.byref(cnt),
            ranks.ctypes.data_as(C.POINTER(C.c_int64)), nrm.ctypes.data_as(C.POINTER(C.c_double)))
        if st == 1 and cnt.value > out_host.numel():  # TT_EINVAL: results larger than the buffer
            out_host = torch.empty(cnt.value, dtype=torch.float64).pin_memory()
            continue
        ctx.check(st)
        return out_host, ranks, nrm, cnt.value
    raise RuntimeError("tt_round_batch_host: output buffer sizing failed")


def tt_sum(ctx: Context, terms, coeffs) -> LibTT:
    arr, keep = _views(terms)
    cf = (C.c_double * len(terms))(*[float(c) for c in coeffs])
    h = C.c_void_p()
    ctx.check(ctx.lib.tt_sum(ctx.handle, len(terms), cf, arr, C.byref(h)))
    return LibTT(ctx, h)


def tt_dot_batch(ctx: Context, xs, ys) -> torch.Tensor:
    P = len(xs)
    out = torch.empty(P, dtype=torch.float64, device=f"cuda:{ctx.device}")
    ax, k1 = _views(xs)
    ay, k2 = _views(ys)
    ctx.check(ctx.lib.tt_dot_batch(ctx.handle, P, ax, ay, C.c_void_p(out.data_ptr())))
    return out


def tt_gram(ctx: Context, tensors) -> torch.Tensor:
    m = len(tensors)
    G = torch.empty((m, m), dtype=torch.float64, device=f"cuda:{ctx.device}")
    arr, keep = _views(tensors)
    ctx.check(ctx.lib.tt_gram(ctx.handle, m, arr, C.c_void_p(G.data_ptr())))
    return G


def tt_gram_blocks(ctx: Context, tensors, blocks: Sequence[Tuple[int, int, int, int]]) -> torch.Tensor:
    m = len(tensors)
    total = sum(bi * bj for _, _, bi, bj in blocks)
    out = torch.empty(max(total, 1), dtype=torch.float64, device=f"cuda:{ctx.device}")
    flat = (C.c_int32 * (4 * len(blocks)))(*[int(v) for b in blocks for v in b])
    arr, keep = _views(tensors)
    ctx.check(ctx.lib.tt_gram_blocks(ctx.handle, m, arr, len(blocks), flat, C.c_void_p(out.data_ptr())))
    return out[:total]


def ttm_device(cores4: Sequence[np.ndarray], device="cuda") -> DeviceTT:
    """A TT-matrix (operator cores (ra_k, n_k, n_k, ra_{k+1})) as the view tt_matvec takes:
    core k reshaped to (ra_k, n_k^2, ra_{k+1}) (row index, then column index)."""
    cs = [np.ascontiguousarray(c, dtype=np.float64) for c in cores4]
    return DeviceTT.from_numpy([c.reshape(c.shape[0], c.shape[1] * c.shape[2], c.shape[3]) for c in cs], device)


def tt_matvec(ctx: Context, A: DeviceTT, x) -> LibTT:
    """y = A x (include/tt_b200.h tt_matvec)."""
    va, ka = A._view()
    vx, kx = x._view()
    h = C.c_void_p()
    ctx.check(ctx.lib.tt_matvec(ctx.handle, C.byref(va), C.byref(vx), C.byref(h)))
    return LibTT(ctx, h)


def laplacian_cores(d: int, n: int) -> List[np.ndarray]:
    """-Delta_d (Dirichlet, unit mesh width: L = tridiag(-1, 2, -1); the 1/h^2 factor cancels in
    the normalised Krylov set) as TT-matrix cores of ranks (1, 2, .., 2, 1): [L I],
    [[I 0], [L I]], .., [I; L] (Kazeev 2012).  DESIGN.md readings A24-A26."""
    L = np.diag(np.full(n, 2.0)) + np.diag(np.full(n - 1, -1.0), 1) + np.diag(np.full(n - 1, -1.0), -1)
    E = np.identity(n)
    if d == 1:
        return [L[None, :, :, None]]
    cores = [np.stack([L, E], axis=-1)[None]]                                  # (1, n, n, 2)
    mid = np.zeros((2, n, n, 2))
    mid[0, :, :, 0], mid[1, :, :, 0], mid[1, :, :, 1] = E, L, E
    cores += [mid.copy() for _ in range(d - 2)]
    cores.append(np.stack([E, L], axis=0)[..., None])                          # (2, n, n, 1)
    return cores


def krylov_set(ctx: Context, d: int, n: int, m: int) -> List[LibTT]:
    """The paper's input sets: a_1 = ones / ||ones||, a_{j+1} = the normalised
    rank-1 TT-rounding (accuracy replaced by maximum rank 1, floor off) of -Delta_d a_j."""
    A = ttm_device(laplacian_cores(d, n), device=f"cuda:{ctx.device}")
    x = DeviceTT.from_numpy([np.ones((1, n, 1)) for _ in range(d)], device=f"cuda:{ctx.device}")
    out: List[LibTT] = []
    for _ in range(m):
        r, _ = tt_round(ctx, [x], [1.0], 0.0, floor_c=0.0, max_rank=1)
        a = tt_sum(ctx, [r], [1.0 / tt_norm(ctx, r)])  # ||round(x)|| (< ||x|| after truncation)
        a.norm = 1.0
        out.append(a)
        x = tt_matvec(ctx, A, a)
    return out


def storage_count(ranks: Sequence[int], modes: Sequence[int]) -> int:
    """Numerator of Eq. (1): sum_k r_{k-1} n_k r_k."""
    return int(sum(ranks[k] * modes[k] * ranks[k + 1] for k in range(len(modes))))


def compression_ratio(ranks: Sequence[int], modes: Sequence[int]) -> float:
    """Eq. (1): TT storage over dense storage."""
    return storage_count(ranks, modes) / float(np.prod(np.asarray(modes, dtype=np.float64)))


def compression_gain(ranks_before: Sequence[int], ranks_after: Sequence[int], modes: Sequence[int]) -> float:
    """Eq. (2): ratio of the compression ratios of x and of its rounding."""
    return storage_count(ranks_before, modes) / float(storage_count(ranks_after, modes))


def tt_element(ctx: Context, x, lin_idx: Sequence[int]) -> torch.Tensor:
    out = torch.empty(len(lin_idx), dtype=torch.float64, device=f"cuda:{ctx.device}")
    v, keep = x._view()
    idx = (C.c_int64 * len(lin_idx))(*[int(i) for i in lin_idx])
    ctx.check(ctx.lib.tt_element(ctx.handle, C.byref(v), len(lin_idx), idx, C.c_void_p(out.data_ptr())))
    return out


def tt_norm(ctx: Context, x) -> float:
    v, keep = x._view()
    o = C.c_double()
    ctx.check(ctx.lib.tt_norm(ctx.handle, C.byref(v), C.byref(o)))
    return o.value


class RoundTrace:
    """Records the TT-sums tt_orth rounds (tt_ctx_round_hook) for the selected call indices
    (Table 1 order, 0-based; None = all): calls[i] = (coeffs, [term cores as numpy], term norms,
    rel_tol, floor_c).  Use as a context manager around tt_orth (step-level replay)."""

    def __init__(self, ctx: Context, select=None):
        self.ctx = ctx
        self.select = None if select is None else set(int(i) for i in select)
        self.calls = {}
        self._fn = N.ROUND_HOOK_FN(self._hook)

    def _hook(self, user, call, K, coeff, terms, opts):
        if self.select is not None and call not in self.select:
            return
        cores, norms = [], []
        for l in range(K):
            v = terms[l]
            cs = []
            for k in range(v.d):
                shp = (int(v.r[k]), int(v.n[k]), int(v.r[k + 1]))
                t = torch.as_tensor(_CoreArray(v.core[k], shp, None), device=f"cuda:{self.ctx.device}")
                cs.append(t.cpu().numpy().copy())
            cores.append(cs)
            norms.append(float(v.norm))
        o = opts[0]
        self.calls[int(call)] = ([float(coeff[l]) for l in range(K)], cores, norms, o.rel_tol, o.floor_c)

    def __enter__(self):
        self.ctx.check(self.ctx.lib.tt_ctx_round_hook(self.ctx.handle, self._fn, None))
        return self

    def __exit__(self, *exc):
        self.ctx.lib.tt_ctx_round_hook(self.ctx.handle, N.ROUND_HOOK_FN(), None)
        return False


def tt_orth(ctx: Context, kind: str, tensors, rel_tol: float, floor_c: float = DEFAULT_FLOOR_C,
            theta: float = 0.5, hh_beta_literal: bool = False, want_loo: bool = False,
            keep_u: bool = False, rank_revealing: bool = True, hh_mask: bool = False):
    m = len(tensors)
    arr, keep = _views(tensors)
    o = N.OrthOpts(_opts(rel_tol, floor_c, 0, theta, rank_revealing), int(hh_beta_literal), int(want_loo),
                   int(hh_mask))
    qs = (C.c_void_p * m)()
    R = np.zeros((m, m), dtype=np.float64)
    ncalls = {"cgs": m, "mgs": m, "cgs2": 2 * m, "mgs2": 2 * m, "gram": m, "householder": 4 * m - 1}[kind]
    loo = (C.c_double * m)()
    ranks = (C.c_int64 * ncalls)()
    us = (C.c_void_p * m)() if keep_u else None
    rep = N.OrthReport(0, -1, C.cast(loo, C.POINTER(C.c_double)) if want_loo else None,
                       C.cast(ranks, C.POINTER(C.c_int64)),
                       C.cast(us, C.POINTER(C.c_void_p)) if keep_u else None)
    st = ctx.lib.tt_orth(ctx.handle, N.KINDS[kind], m, arr, C.byref(o), qs,
                         R.ctypes.data_as(C.POINTER(C.c_double)), C.byref(rep))
    if st != 0:
        err = N.TTError(st, ctx.lib.tt_last_error(ctx.handle).decode())
        err.fail_index = rep.fail_index
        raise err
    Q = [LibTT(ctx, C.c_void_p(qs[i])) for i in range(m)]
    report = {"rounding_calls": rep.rounding_calls, "max_rank_per_call": list(ranks[:rep.rounding_calls]),
              "loo_per_step": np.array(loo[:m]) if want_loo else None}
    if keep_u:
        report["u"] = [LibTT(ctx, C.c_void_p(us[i])) if us[i] else None for i in range(m)]
    return Q, R, report
