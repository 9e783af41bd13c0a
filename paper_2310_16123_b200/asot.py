"""Thin Python binding over libasot.so (C ABI: include/asot.h).

Argument marshalling only: torch tensors provide device memory and streams, every step of
the path (mapping, histograms, Gibbs kernel, Sinkhorn, cost, mirroring) runs in the library's
CUDA kernels.  Names follow the ABI / the paper: H is the N x K matrix of mapped marginals
(a' rows), cost is C_s, eps and iters are the Sinkhorn settings.
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib

FP32 = 0  # ASOT_PREC_FP32: fp32-accurate -- 3xTF32 tcgen05 (K >= 32), fp32 CUDA cores (K < 32);
          # rel. err <= 1e-4 target
TF32 = 1  # ASOT_PREC_TF32: tcgen05 kind::tf32 MMA, fp32 accumulate (rel. err <= 2e-3 target)
TILE_SLOTS = 128

FLAG_EMPTY_DIST = 1
FLAG_BAD_MASS = 2
FLAG_NONFINITE_INPUT = 4
FLAG_DENOM_CLAMPED = 8
FLAG_NONFINITE_OUTPUT = 16
FLAG_SOFT_FALLBACK = 32
FLAG_EXACT_TOO_LARGE = 64
FLAG_BAD_INDEX = 128

_STATUS_EXC = {1: ValueError, 2: ValueError, 3: FloatingPointError, 4: RuntimeError,
               5: NotImplementedError, 6: MemoryError}


class AsotStatusError(RuntimeError):
    pass


def _lib_handle():
    return _lib.load()


def _check(rc: int) -> None:
    if rc != 0:
        msg = _lib_handle().asot_last_error().decode()
        raise _STATUS_EXC.get(rc, RuntimeError)(f"asot status {rc}: {msg}")


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        if not t.is_contiguous():
            raise ValueError("tensors must be contiguous")
        return t.data_ptr()
    if isinstance(t, np.ndarray):
        if not t.flags["C_CONTIGUOUS"]:
            raise ValueError("arrays must be C-contiguous")
        return t.ctypes.data
    raise TypeError(type(t))


def _stream(stream) -> Optional[int]:
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


def _need_cuda(*ts):
    for t in ts:
        if t is not None and (not isinstance(t, torch.Tensor) or not t.is_cuda):
            raise ValueError("device tensors (cuda) are required; there is no CPU path")


def _need_f32(*ts):
    for t in ts:
        if t is not None and t.dtype != torch.float32:
            raise ValueError(f"float32 tensors are required (got {t.dtype})")


def _pair_list(pair_i, pair_j) -> int:
    """Explicit pair lists are two 1-D int32 device tensors of one length (the ABI reads i32:
    an int64 tensor would be read as (low, high) word pairs).  Returns the length."""
    for t in (pair_i, pair_j):
        if t.dtype != torch.int32:
            raise ValueError(f"pair_i / pair_j must be int32 tensors (got {t.dtype})")
        if t.dim() != 1:
            raise ValueError("pair_i / pair_j must be 1-D")
    if pair_i.numel() != pair_j.numel():
        raise ValueError(f"pair_i has {pair_i.numel()} entries, pair_j {pair_j.numel()}")
    return int(pair_i.numel())


def _hist_cost(H, cost):
    """H [N, K] and C_s [K, K], both f32."""
    _need_f32(H, cost)
    if H.dim() != 2 or cost.dim() != 2 or cost.shape[0] != cost.shape[1] or cost.shape[0] != H.shape[1]:
        raise ValueError(f"need H [N, K] and cost [K, K] (got {tuple(H.shape)}, {tuple(cost.shape)})")


def num_tiles(n_dist: int) -> int:
    return int(_lib_handle().asot_num_tiles(int(n_dist)))


def effective_precision(n_anchors: int, precision: int) -> int:
    return int(_lib_handle().asot_effective_precision(int(n_anchors), int(precision)))


KERNEL_NAMES = {0: "sinkhorn_simt_kernel (fp32 CUDA cores)",
                1: "sinkhorn_tc_kernel (TF32, 1 SM, M=128)",
                2: "sinkhorn_tc2_kernel (TF32, CTA pair, cta_group::2, M=256)",
                3: "sinkhorn_tc3_kernel (3xTF32 fp32-accurate, 1 SM, M=128)",
                4: "sinkhorn_tc4_kernel (TF32, streamed GEMM form, CTA pair, M=N=256)",
                5: "sinkhorn_tc5_kernel (3xTF32 fp32-accurate, streamed GEMM form, CTA pair, M=N=256)",
                6: "sinkhorn_tc5_kernel (TF32 one-pass, streamed GEMM form, pair-list mode, CTA pair)",
                7: "sinkhorn_tc_kernel (TF32, 1 SM, M=128, pair-list mode)",
                8: "sinkhorn_tc3_kernel (3xTF32 fp32-accurate, 1 SM, M=128, pair-list mode)",
                9: "sinkhorn_warp_kernel (fp32 CUDA cores, lane per anchor, K < 32)",
                10: "sinkhorn_tc6_kernel (BF16x3 fp32-accurate, resident, CTA pair, cta_group::2, M=256)",
                11: "sinkhorn_sparse_rect_kernel<R, C> per support-class pair + the 9-16-bin half-warp form (fp32 CUDA cores, thread per pair, support-ordered; histogram supports <= 16)"}


def sinkhorn_path_kind(H: torch.Tensor, precision: int) -> int:
    """The kernel a call on histograms H [N, K] runs (asot_sinkhorn_path_kind): 11 = the
    small-support kernel, else sinkhorn_kernel_kind(K, precision)."""
    max_support = int((H != 0).sum(dim=1).max().item()) if H.numel() else 0
    return int(_lib_handle().asot_sinkhorn_path_kind(int(H.shape[1]), int(precision), max_support))


def sinkhorn_kernel_kind(n_anchors: int, precision: int) -> int:
    """0 SIMT fp32, 1 TF32 1-SM, 2 TF32 CTA pair, 3 3xTF32 1-SM, 4 TF32 streamed, 5 3xTF32
    streamed (see asot.h)."""
    return int(_lib_handle().asot_sinkhorn_kernel_kind(int(n_anchors), int(precision)))


def last_launch_count() -> int:
    return int(_lib_handle().asot_last_launch_count())


def profile_enable(on: bool = True) -> None:
    """Time every Sinkhorn kernel launch with CUDA events on its launch stream (this thread)."""
    _check(_lib_handle().asot_profile_enable(int(bool(on))))


PROF_SINKHORN = 0
PROF_MAP = 1


def profile_read(reset: bool = True, kernel: int = PROF_SINKHORN) -> tuple[float, int]:
    """(summed kernel milliseconds, launches) since the last reset, for the Sinkhorn kernel
    (PROF_SINKHORN) or the mapping kernel (PROF_MAP)."""
    ms = ctypes.c_double(0.0)
    n = ctypes.c_int64(0)
    _check(_lib_handle().asot_profile_read_kernel(int(kernel), ctypes.byref(ms), ctypes.byref(n),
                                                  int(bool(reset))))
    return float(ms.value), int(n.value)


def profile_clock(kind: int) -> float:
    """Effective SM clock (MHz) of the last launch of Sinkhorn kernel `kind` (in-kernel
    %clock64 / %globaltimer probe; see asot_profile_clock)."""
    mhz = ctypes.c_double(0.0)
    _check(_lib_handle().asot_profile_clock(int(kind), ctypes.byref(mhz)))
    return float(mhz.value)


def new_status(device=None) -> torch.Tensor:
    return torch.zeros(1, dtype=torch.int32, device=device or "cuda")


def check_status(status, allow: int = FLAG_DENOM_CLAMPED | FLAG_SOFT_FALLBACK | FLAG_EXACT_TOO_LARGE) -> int:
    """Raise on data-dependent failures the kernels flagged (call after synchronising)."""
    v = int(status.item()) if isinstance(status, torch.Tensor) else int(status)
    bad = v & ~allow
    if bad & (FLAG_EMPTY_DIST | FLAG_BAD_MASS):
        raise ValueError(f"infeasible mass (status flags {v:#x})")
    if bad & FLAG_BAD_INDEX:
        raise ValueError(f"pair-list index outside [0, n_dist) (status flags {v:#x})")
    if bad & (FLAG_NONFINITE_INPUT | FLAG_NONFINITE_OUTPUT):
        raise FloatingPointError(f"non-finite values (status flags {v:#x})")
    return v


class Workspace:
    """Caller-owned device scratch (grown on demand, reused across calls)."""

    def __init__(self, device=None):
        self.device = device or "cuda"
        self.buf = torch.empty(0, dtype=torch.uint8, device=self.device)

    def get(self, nbytes: int) -> torch.Tensor:
        if self.buf.numel() < nbytes:
            self.buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=self.device)
        return self.buf


_default_ws = {}


def _ws(workspace: Optional[Workspace], device) -> Workspace:
    if workspace is not None:
        return workspace
    key = str(device)
    if key not in _default_ws:
        _default_ws[key] = Workspace(device)
    return _default_ws[key]


def _host_offsets(offsets, offsets_host):
    if offsets_host is not None:
        return np.ascontiguousarray(offsets_host, dtype=np.int64)
    return np.ascontiguousarray(offsets.detach().cpu().numpy(), dtype=np.int64)


def _map_ws_call(points, offsets, oh, weights, N, d, anchors, K, assign, H, peer_ptrs, row_base, st,
                 workspace, stream):
    """asot_map_to_anchors_ws: the mapping with the tensor-core score pass (same bits out)."""
    lib = _lib_handle()
    need = int(lib.asot_map_workspace_bytes(int(oh[-1]), int(K)))
    buf = _ws(workspace, points.device).get(need)
    _check(lib.asot_map_to_anchors_ws(
        _ptr(points), _ptr(offsets), _ptr(oh), _ptr(weights), N, int(d), _ptr(anchors), int(K),
        _ptr(assign), _ptr(H), _ptr(peer_ptrs) if peer_ptrs is not None else None,
        int(peer_ptrs.numel()) if peer_ptrs is not None else 0, int(row_base), _ptr(st), _ptr(buf),
        int(buf.numel()), _stream(stream)))


def map_to_anchors(points: torch.Tensor, offsets: torch.Tensor, weights: torch.Tensor,
                   anchors: torch.Tensor, offsets_host: Optional[np.ndarray] = None,
                   status: Optional[torch.Tensor] = None, stream=None, tensor_core: bool = False,
                   workspace: Optional[Workspace] = None):
    """Steps a2 + a3: returns (assign [T] int32, H [N, K] f32, status).  tensor_core=True:
    asot_map_to_anchors_ws (score products on tcgen05, bit-identical results)."""
    _need_cuda(points, offsets, weights, anchors)
    _need_f32(points, weights, anchors)
    oh = _host_offsets(offsets, offsets_host)
    N = oh.shape[0] - 1
    T = int(oh[-1])
    K, d = anchors.shape
    assign = torch.empty(max(T, 1), dtype=torch.int32, device=points.device)
    H = torch.empty((N, K), dtype=torch.float32, device=points.device)
    st = new_status(points.device) if status is None else status
    if tensor_core:
        _map_ws_call(points, offsets, oh, weights, N, d, anchors, K, assign, H, None, 0, st, workspace,
                     stream)
        return assign[:T], H, st
    _check(_lib_handle().asot_map_to_anchors(
        _ptr(points), _ptr(offsets), _ptr(oh), _ptr(weights), N, int(d), _ptr(anchors), int(K),
        _ptr(assign), _ptr(H), _ptr(st), _stream(stream)))
    return assign[:T], H, st


def map_to_anchors_bcast(points: torch.Tensor, offsets: torch.Tensor, weights: torch.Tensor,
                         anchors: torch.Tensor, peer_ptrs: torch.Tensor, row_base: int,
                         offsets_host: Optional[np.ndarray] = None,
                         status: Optional[torch.Tensor] = None, stream=None,
                         tensor_core: bool = False, workspace: Optional[Workspace] = None):
    """map_to_anchors that also stores each H row into every matrix of `peer_ptrs` (int64 device
    tensor of device addresses of full [N_total, K] H buffers) at row row_base + i."""
    _need_cuda(points, offsets, weights, anchors, peer_ptrs)
    _need_f32(points, weights, anchors)
    oh = _host_offsets(offsets, offsets_host)
    N = oh.shape[0] - 1
    T = int(oh[-1])
    K, d = anchors.shape
    assign = torch.empty(max(T, 1), dtype=torch.int32, device=points.device)
    H = torch.empty((N, K), dtype=torch.float32, device=points.device)
    st = new_status(points.device) if status is None else status
    if tensor_core:
        _map_ws_call(points, offsets, oh, weights, N, d, anchors, K, assign, H, peer_ptrs, row_base, st,
                     workspace, stream)
        return assign[:T], H, st
    _check(_lib_handle().asot_map_to_anchors_bcast(
        _ptr(points), _ptr(offsets), _ptr(oh), _ptr(weights), N, int(d), _ptr(anchors), int(K),
        _ptr(assign), _ptr(H), _ptr(peer_ptrs), int(peer_ptrs.numel()), int(row_base), _ptr(st),
        _stream(stream)))
    return assign[:T], H, st


def _soft_common(points, offsets, weights, offsets_host, K, status, want_codes):
    _need_cuda(points, offsets, weights)
    oh = _host_offsets(offsets, offsets_host)
    N = oh.shape[0] - 1
    T = int(oh[-1])
    H = torch.empty((N, K), dtype=torch.float32, device=points.device)
    codes = torch.empty((max(T, 1), K), dtype=torch.float32, device=points.device) if want_codes else None
    st = new_status(points.device) if status is None else status
    return oh, N, T, H, codes, st


def map_soft_ml(points: torch.Tensor, offsets: torch.Tensor, weights: torch.Tensor,
                W1: torch.Tensor, b1: torch.Tensor, W2: torch.Tensor, b2: torch.Tensor,
                offsets_host: Optional[np.ndarray] = None, want_codes: bool = False,
                status: Optional[torch.Tensor] = None, workspace: Optional[Workspace] = None,
                tensor_cores: bool = True, stream=None):
    """NEXT-1 ASOT-ML mapping: codes |MLP(x)| / l1 and H = Z^T a per distribution.
    ``tensor_cores=False`` passes no workspace, which selects the CUDA-core kernel (the
    cross-check implementation).  Returns (H [N, K], codes [T, K] or None, status)."""
    _need_cuda(W1, b1, W2, b2)
    _need_f32(points, weights, W1, b1, W2, b2)
    d, hidden = W1.shape
    K = int(W2.shape[1])
    if tuple(b1.shape) != (hidden,) or tuple(W2.shape) != (hidden, K) or tuple(b2.shape) != (K,):
        raise ValueError("ML weights: W1 [d, h], b1 [h], W2 [h, K], b2 [K]")
    oh, N, T, H, codes, st = _soft_common(points, offsets, weights, offsets_host, K, status, want_codes)
    L = _lib_handle()
    nbytes = int(L.asot_map_soft_ml_workspace_bytes(int(d), int(hidden), K)) if tensor_cores else 0
    ws = _ws(workspace, points.device).get(nbytes) if nbytes > 0 else None
    _check(L.asot_map_soft_ml(
        _ptr(points), _ptr(offsets), _ptr(oh), _ptr(weights), N, int(d), K, int(hidden), _ptr(W1),
        _ptr(b1), _ptr(W2), _ptr(b2), _ptr(H), _ptr(codes), _ptr(st), _ptr(ws),
        0 if ws is None else ws.numel(), _stream(stream)))
    return H, (codes[:T] if codes is not None else None), st


def map_soft_dl(points: torch.Tensor, offsets: torch.Tensor, weights: torch.Tensor,
                dictionary: torch.Tensor, V1: torch.Tensor, c1: torch.Tensor, v2: torch.Tensor,
                c2: torch.Tensor, n_layers: int = 20, offsets_host: Optional[np.ndarray] = None,
                want_codes: bool = False, status: Optional[torch.Tensor] = None,
                workspace: Optional[Workspace] = None, stream=None):
    """NEXT-1 ASOT-DL near-one-hot encoder (Eq. (9), L layers) and H = Z^T a per distribution.
    Returns (H [N, K], codes [T, K] or None, status)."""
    _need_cuda(dictionary, V1, c1, v2, c2)
    _need_f32(points, weights, dictionary, V1, c1, v2, c2)
    K, d = dictionary.shape
    hidden = int(V1.shape[1])
    oh, N, T, H, codes, st = _soft_common(points, offsets, weights, offsets_host, int(K), status,
                                          want_codes)
    L = _lib_handle()
    nbytes = int(L.asot_map_soft_dl_workspace_bytes(int(d), int(K), int(T)))
    ws = _ws(workspace, points.device).get(nbytes) if nbytes > 0 else None
    _check(L.asot_map_soft_dl(
        _ptr(points), _ptr(offsets), _ptr(oh), _ptr(weights), N, int(d), _ptr(dictionary), int(K),
        int(n_layers), hidden, _ptr(V1), _ptr(c1), _ptr(v2), _ptr(c2), _ptr(H), _ptr(codes),
        _ptr(st), _ptr(ws), 0 if ws is None else ws.numel(), _stream(stream)))
    return H, (codes[:T] if codes is not None else None), st


def mahalanobis_cost(anchors: torch.Tensor, M: torch.Tensor, normalize: bool = True,
                     workspace: Optional[Workspace] = None, stream=None) -> torch.Tensor:
    """ASOT-ML anchor cost C_s[u, v] = ||M w_u - M w_v||_2, optionally / max."""
    _need_cuda(anchors, M)
    _need_f32(anchors, M)
    K, d = anchors.shape
    h = int(M.shape[0])
    C = torch.empty((K, K), dtype=torch.float32, device=anchors.device)
    L = _lib_handle()
    ws = _ws(workspace, anchors.device).get(L.asot_mahalanobis_workspace_bytes(int(K), h))
    _check(L.asot_mahalanobis_cost(_ptr(anchors), int(K), int(d), _ptr(M), h, int(bool(normalize)),
                                   _ptr(C), _ptr(ws), ws.numel(), _stream(stream)))
    return C


def kmeans_minibatch(points: torch.Tensor, init_centers: torch.Tensor, batch_idx: torch.Tensor,
                     status: Optional[torch.Tensor] = None, stream=None):
    """NEXT-2 ASOT-k anchor learning: mini-batch k-means.  batch_idx [iters, b]
    int64 point indices (the random draws).  Returns (centers f64 [K, d], anchors f32 [K, d],
    counts i64 [K], status)."""
    _need_cuda(points, init_centers, batch_idx)
    _need_f32(points)
    if batch_idx.dtype != torch.int64:
        raise ValueError("batch_idx must be int64")
    T, d = points.shape
    K = int(init_centers.shape[0])
    iters, b = batch_idx.shape
    centers = init_centers.to(torch.float64).contiguous().clone()
    counts = torch.zeros(K, dtype=torch.int64, device=points.device)
    anchors = torch.empty((K, d), dtype=torch.float32, device=points.device)
    assign = torch.empty(max(int(b), 1), dtype=torch.int32, device=points.device)
    st = new_status(points.device) if status is None else status
    _check(_lib_handle().asot_kmeans_minibatch(
        _ptr(points), int(T), int(d), K, _ptr(batch_idx), int(b), int(iters),
        _ptr(centers), _ptr(counts), _ptr(anchors), _ptr(assign), _ptr(st), _stream(stream)))
    return centers, anchors, counts, st


def sqeuclid_cost(anchors: torch.Tensor, normalize: bool = True, stream=None) -> torch.Tensor:
    """C_s[u, v] = ||w_u - w_v||^2 (/ max) of device anchors (R#7)."""
    _need_cuda(anchors)
    _need_f32(anchors)
    K, d = anchors.shape
    C = torch.empty((K, K), dtype=torch.float32, device=anchors.device)
    _check(_lib_handle().asot_sqeuclid_cost(_ptr(anchors), int(K), int(d), int(bool(normalize)),
                                            _ptr(C), _stream(stream)))
    return C


def eot_pairs(points: torch.Tensor, offsets: torch.Tensor, weights: torch.Tensor,
              pair_i: torch.Tensor, pair_j: torch.Tensor, eps: float, iters: int,
              cost_scale: float, offsets_host: Optional[np.ndarray] = None,
              status: Optional[torch.Tensor] = None, workspace: Optional[Workspace] = None,
              stream=None) -> torch.Tensor:
    """NEXT-4 baseline: entropic OT on the original point sets for explicit pairs (ground cost
    cost_scale * ||x - y||^2).  Returns dist [n_pairs] f32."""
    _need_cuda(points, offsets, weights, pair_i, pair_j)
    _need_f32(points, weights)
    n = _pair_list(pair_i, pair_j)
    if n == 0:
        return torch.empty(0, dtype=torch.float32, device=points.device)
    oh = _host_offsets(offsets, offsets_host)
    N = oh.shape[0] - 1
    out = torch.empty(max(n, 1), dtype=torch.float32, device=points.device)
    st = new_status(points.device) if status is None else status
    L = _lib_handle()
    ws = _ws(workspace, points.device).get(L.asot_eot_workspace_bytes(N, _ptr(oh), n))
    _check(L.asot_eot_pairs(_ptr(points), _ptr(offsets), _ptr(oh), _ptr(weights), N,
                            int(points.shape[1]), float(cost_scale), float(eps), int(iters),
                            _ptr(pair_i), _ptr(pair_j), n, _ptr(out), _ptr(st), _ptr(ws),
                            ws.numel(), _stream(stream)))
    return out[:n]


def exact_asot_pairs(H: torch.Tensor, cost: torch.Tensor, pair_i: torch.Tensor, pair_j: torch.Tensor,
                     status: Optional[torch.Tensor] = None, workspace: Optional[Workspace] = None,
                     stream=None) -> torch.Tensor:
    """NEXT-3: exact anchor-space OT W_AS for explicit pairs (fp64 min-cost flow on the histogram
    supports; a warp per pair up to 128-bin supports, a CTA per pair above).  Returns dist [n_pairs]
    f64 (NaN for invalid indices or an empty support)."""
    _hist_cost(H, cost)
    n = _pair_list(pair_i, pair_j)
    _need_cuda(H, cost, pair_i, pair_j)
    if n == 0:
        return torch.empty(0, dtype=torch.float64, device=H.device)
    N, K = H.shape
    out = torch.empty(max(n, 1), dtype=torch.float64, device=H.device)
    st = new_status(H.device) if status is None else status
    ws = _ws(workspace, H.device).get(int(_lib_handle().asot_exact_asot_workspace_bytes(n, int(K))))
    _check(_lib_handle().asot_exact_asot_pairs(_ptr(H), N, int(K), _ptr(cost), _ptr(pair_i), _ptr(pair_j),
                                               n, _ptr(out), _ptr(st), _ptr(ws), ws.numel(), _stream(stream)))
    return out[:n]


def exact_w1_points(points: torch.Tensor, offsets: torch.Tensor, weights: torch.Tensor,
                    pair_i: torch.Tensor, pair_j: torch.Tensor, status: Optional[torch.Tensor] = None,
                    stream=None) -> torch.Tensor:
    """NEXT-3 bound checks: exact W_1 on the original point sets with the Euclidean ground metric
    (supports <= 64 points per side; larger: NaN + FLAG_EXACT_TOO_LARGE).  Returns [n_pairs] f64."""
    _need_f32(points, weights)
    n = _pair_list(pair_i, pair_j)
    _need_cuda(points, offsets, weights, pair_i, pair_j)
    out = torch.empty(n, dtype=torch.float64, device=points.device)
    if n == 0:
        return out
    st = new_status(points.device) if status is None else status
    _check(_lib_handle().asot_exact_w1_points(_ptr(points), _ptr(offsets), _ptr(weights),
                                              int(offsets.numel()) - 1, int(points.shape[1]), _ptr(pair_i),
                                              _ptr(pair_j), n, _ptr(out), _ptr(st), _stream(stream)))
    return out


def bound_terms(points: torch.Tensor, offsets: torch.Tensor, anchors: torch.Tensor, assign: torch.Tensor,
                cost: torch.Tensor, pair_i: torch.Tensor, pair_j: torch.Tensor,
                status: Optional[torch.Tensor] = None, stream=None):
    """NEXT-3: per pair (Prop. 1 ||C_hat - C||_1, max |C_hat - C|, Prop. 2 residual bound), each
    [n_pairs] f64, for the one-hot assignments `assign` and the anchor cost `cost` (C_s of W_AS)."""
    _need_f32(points, anchors, cost)
    if assign.dtype != torch.int32:
        raise ValueError("assign must be int32")
    n = _pair_list(pair_i, pair_j)
    _need_cuda(points, offsets, anchors, assign, cost, pair_i, pair_j)
    outs = [torch.empty(n, dtype=torch.float64, device=points.device) for _ in range(3)]
    if n == 0:
        return tuple(outs)
    st = new_status(points.device) if status is None else status
    _check(_lib_handle().asot_bound_terms(_ptr(points), _ptr(offsets), int(offsets.numel()) - 1,
                                          int(points.shape[1]), _ptr(anchors), int(anchors.shape[0]),
                                          _ptr(assign), _ptr(cost), _ptr(pair_i), _ptr(pair_j), n,
                                          _ptr(outs[0]), _ptr(outs[1]), _ptr(outs[2]), _ptr(st),
                                          _stream(stream)))
    return tuple(outs)


def pairwise_sinkhorn(H: torch.Tensor, cost: torch.Tensor, eps: float, iters: int,
                      pair_i: torch.Tensor, pair_j: torch.Tensor, precision: int = TF32,
                      cost_max: Optional[float] = None, status: Optional[torch.Tensor] = None,
                      workspace: Optional[Workspace] = None, stream=None) -> torch.Tensor:
    """Steps a1 + a5 + a6 on explicit pairs (a = H[pair_i] on the u side).  pair_i / pair_j:
    int32 device tensors of one length; an entry outside [0, N) gives NaN and FLAG_BAD_INDEX."""
    _hist_cost(H, cost)
    n = _pair_list(pair_i, pair_j)
    _need_cuda(H, cost, pair_i, pair_j)
    if n == 0:
        return torch.empty(0, dtype=torch.float32, device=H.device)
    N, K = H.shape
    out = torch.empty(n, dtype=torch.float32, device=H.device)
    cmax = float(cost.max().item()) if cost_max is None else float(cost_max)
    st = new_status(H.device) if status is None else status
    L = _lib_handle()
    ws = _ws(workspace, H.device).get(L.asot_pairwise_list_workspace_bytes(int(N), int(K), int(precision),
                                                                           int(n)))
    _check(L.asot_pairwise_sinkhorn(
        _ptr(H), N, int(K), _ptr(cost), cmax, float(eps), int(iters), int(precision),
        _ptr(pair_i), _ptr(pair_j), n, _ptr(out), _ptr(st), _ptr(ws), ws.numel(), _stream(stream)))
    return out


def distance_matrix(points: Optional[torch.Tensor], offsets: Optional[torch.Tensor],
                    weights: Optional[torch.Tensor], anchors: Optional[torch.Tensor],
                    cost: torch.Tensor, eps: float, iters: int, precision: int = TF32,
                    hist: Optional[torch.Tensor] = None, n_dist: Optional[int] = None,
                    tile_range: Optional[Sequence[int]] = None, out: Optional[torch.Tensor] = None,
                    packed: Optional[torch.Tensor] = None, want_matrix: bool = True,
                    assign_out: Optional[torch.Tensor] = None, hist_out: Optional[torch.Tensor] = None,
                    offsets_host: Optional[np.ndarray] = None, cost_max: Optional[float] = None,
                    status: Optional[torch.Tensor] = None, workspace: Optional[Workspace] = None,
                    stream=None, out_ptr: Optional[int] = None):
    """Full pipeline a1-a6.  Returns the N x N matrix (when want_matrix) and/or fills `packed`
    ([(tile_end - tile_begin) * 128] slot-ordered results) for the tile range.  `out_ptr` (with
    want_matrix=False) is a raw device address of an N x N f32 matrix to write the range's pairs
    into -- e.g. a peer GPU's symmetric-memory buffer, so the results travel as NVLink stores
    straight from the Sinkhorn epilogue (distributed.py)."""
    _need_cuda(cost, hist, points, offsets, weights, anchors)
    _need_f32(cost, hist, points, weights, anchors)
    L = _lib_handle()
    K = int(cost.shape[0])
    if hist is None:
        oh = _host_offsets(offsets, offsets_host)
        N = oh.shape[0] - 1
        T = int(oh[-1])
        d = int(points.shape[1])
        dev = points.device
    else:
        oh = None
        N = int(hist.shape[0]) if n_dist is None else int(n_dist)
        T, d = 0, 1
        dev = hist.device
    nt = num_tiles(N)
    t0, t1 = (0, nt) if tile_range is None else (int(tile_range[0]), int(tile_range[1]))
    if want_matrix and out is None:
        out = torch.empty((N, N), dtype=torch.float32, device=dev)
    if not want_matrix:
        out = None
    cmax = float(cost.max().item()) if cost_max is None else float(cost_max)
    st = new_status(dev) if status is None else status
    ws = _ws(workspace, dev).get(L.asot_distance_matrix_workspace_bytes(N, T, K, int(precision)))
    out_addr = _ptr(out) if out is not None else out_ptr
    _check(L.asot_distance_matrix(
        _ptr(points), _ptr(offsets), _ptr(oh), _ptr(weights), N, d, _ptr(anchors), K, _ptr(cost),
        cmax, float(eps), int(iters), int(precision), _ptr(hist), t0, t1, out_addr, _ptr(packed),
        _ptr(assign_out), _ptr(hist_out), _ptr(st), _ptr(ws), ws.numel(), _stream(stream)))
    return out


def distance_matrix_partition(hist: torch.Tensor, cost: torch.Tensor, eps: float, iters: int,
                              part: Sequence[int], precision: int = TF32,
                              out: Optional[torch.Tensor] = None, out_ptr: Optional[int] = None,
                              cost_max: Optional[float] = None, status: Optional[torch.Tensor] = None,
                              workspace: Optional[Workspace] = None, stream=None):
    """asot_distance_matrix_partition: part (p0, p1) of the pair enumeration the call picks
    (support order on the small-support path, the a4 tiles otherwise), results into `out` [N, N]
    or the raw device address `out_ptr` (e.g. a peer GPU's symmetric-memory matrix); a partition
    of [0, num_tiles(N)) over calls covers every pair once.  Returns `out`."""
    _hist_cost(hist, cost)
    _need_cuda(hist, cost)
    L = _lib_handle()
    N, K = int(hist.shape[0]), int(hist.shape[1])
    if out is None and out_ptr is None:
        out = torch.empty((N, N), dtype=torch.float32, device=hist.device)
    cmax = float(cost.max().item()) if cost_max is None else float(cost_max)
    st = new_status(hist.device) if status is None else status
    ws = _ws(workspace, hist.device).get(L.asot_distance_matrix_workspace_bytes(N, 0, K, int(precision)))
    _check(L.asot_distance_matrix_partition(
        _ptr(hist), N, K, _ptr(cost), cmax, float(eps), int(iters), int(precision), int(part[0]),
        int(part[1]), _ptr(out) if out is not None else out_ptr, _ptr(st), _ptr(ws), ws.numel(),
        _stream(stream)))
    return out


def host_workspace_bytes(n_dist: int, n_points: int, dim: int, n_anchors: int,
                         precision: int = TF32) -> int:
    return int(_lib_handle().asot_distance_matrix_host_workspace_bytes(
        int(n_dist), int(n_points), int(dim), int(n_anchors), int(precision)))


def distance_matrix_host(points: np.ndarray, offsets: np.ndarray, weights: np.ndarray,
                         anchors: np.ndarray, cost: np.ndarray, eps: float, iters: int,
                         precision: int = TF32, out: Optional[np.ndarray] = None,
                         workspace: Optional[Workspace] = None, device=None, stream=None):
    """End to end from host buffers (H2D copies, the whole pipeline, D2H of the matrix) through
    the single C-ABI call asot_distance_matrix_host.  Returns (D [N, N] host f32, status)."""
    pts = np.ascontiguousarray(points, dtype=np.float32)
    offs = np.ascontiguousarray(offsets, dtype=np.int64)
    w = np.ascontiguousarray(weights, dtype=np.float32)
    anc = np.ascontiguousarray(anchors, dtype=np.float32)
    cst = np.ascontiguousarray(cost, dtype=np.float32)
    N = offs.shape[0] - 1
    K, d = anc.shape
    if out is None:
        out = np.empty((N, N), dtype=np.float32)
    status = np.zeros(1, dtype=np.uint32)
    dev = device or torch.device("cuda", torch.cuda.current_device())
    L = _lib_handle()
    ws = _ws(workspace, dev).get(host_workspace_bytes(N, pts.shape[0], d, K, precision))
    _check(L.asot_distance_matrix_host(
        _ptr(pts), _ptr(offs), _ptr(w), N, int(d), _ptr(anc), int(K), _ptr(cst), float(eps),
        int(iters), int(precision), _ptr(out), _ptr(status), _ptr(ws), ws.numel(), _stream(stream)))
    return out, int(status[0])


def tile_pairs(n_dist: int, tile_begin: int = 0, tile_end: Optional[int] = None):
    """Host enumeration of the tile slots: returns (i, j, valid) numpy arrays."""
    t1 = num_tiles(n_dist) if tile_end is None else int(tile_end)
    n = (t1 - int(tile_begin)) * TILE_SLOTS
    i = np.empty(n, np.int32)
    j = np.empty(n, np.int32)
    v = np.empty(n, np.uint8)
    _check(_lib_handle().asot_tile_pairs_host(int(n_dist), int(tile_begin), t1, _ptr(i), _ptr(j), _ptr(v)))
    return i, j, v.astype(bool)


def unpack_tiles(packed: torch.Tensor, n_dist: int, tile_begin: int, tile_end: int,
                 out: torch.Tensor, zero_diag: bool = True, stream=None) -> torch.Tensor:
    """KN6: scatter slot-ordered tile results into the N x N matrix (both triangles)."""
    _need_cuda(packed, out)
    _check(_lib_handle().asot_unpack_tiles(_ptr(packed), int(n_dist), int(tile_begin),
                                           int(tile_end), _ptr(out), int(bool(zero_diag)),
                                           _stream(stream)))
    return out
