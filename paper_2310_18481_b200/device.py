"""ctypes binding of the C-ABI library ``libmosel_b200.so``.

This is the same binding a maintainer of the reference would add (see
INTEGRATION.md): plain pointers and sizes, a ``cudaStream_t`` per call, an
``int`` status mapped to ``ValueError`` subclasses.  PyTorch provides device
memory and the current stream only.  There is no fallback: if the library
or a CUDA device is missing, every entry point raises.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "libmosel_b200.so"
GEMM_PLAN_BYTES = 2048
OP_BYTES = 2112
DROP = -1
MS_ERR_CUDA_STATUS = 2

_lib = None


class DeviceError(ValueError):
    """A C-ABI call returned a nonzero status."""


SEG_NO_RELU = 1


class Segment(C.Structure):
    _fields_ = [("n_begin", C.c_int), ("n_end", C.c_int), ("ptr", C.c_void_p),
                ("ldd", C.c_longlong), ("col0", C.c_int), ("flags", C.c_int)]


class RowDesc(C.Structure):
    _fields_ = [("lines", C.c_longlong), ("width", C.c_int), ("c_src", C.c_int), ("c_dst", C.c_int),
                ("pad_w", C.c_int), ("src_u8", C.c_int), ("u8_scale", C.c_float), ("u8_bias", C.c_float),
                ("frame_h", C.c_int), ("pad_h", C.c_int), ("slot_off", C.c_int), ("plane_stride", C.c_longlong)]


_P, _I, _LL, _D = C.c_void_p, C.c_int, C.c_longlong, C.c_double

PASS_MAX_K, PASS_MAX_PTS, PASS_MAX_MEMBERS = 8, 32, 1024
PASS_SUMMARY = 2 + PASS_MAX_K


class PassCost(C.Structure):
    """MsPassCost: integer pass-time model of ms_pass_select (mosel_b200.h)."""
    _fields_ = [("K", C.c_int), ("n_pts", C.c_int), ("w", C.c_int32 * PASS_MAX_K),
                ("u", C.c_int64 * PASS_MAX_PTS), ("t_ns", C.c_int64 * PASS_MAX_PTS)]

    @classmethod
    def make(cls, w, u, t_ns):
        c = cls()
        c.K, c.n_pts = len(w), len(u)
        if not (1 <= c.K <= PASS_MAX_K and 1 <= c.n_pts <= PASS_MAX_PTS and len(t_ns) == c.n_pts):
            raise ValueError("PassCost: K in 1..8, 1..32 knots")
        for i, v in enumerate(w):
            c.w[i] = int(v)
        for i, (a, b) in enumerate(zip(u, t_ns)):
            c.u[i], c.t_ns[i] = int(a), int(b)
        return c

    def table(self):
        """(w, u, t_ns) as Python int lists (the oracle's arguments)."""
        return (list(self.w[: self.K]), list(self.u[: self.n_pts]), list(self.t_ns[: self.n_pts]))
_SIGS = {
    "ms_abi_version": ([], C.c_int),
    "ms_set_pdl": ([_I], C.c_int),
    "ms_set_occ2_grid": ([_I], C.c_int),
    "ms_strategy_dp": ([_I, _P, _P, _P, _I, _I, _P, _P, _P], C.c_int),
    "ms_policy_apply": ([_I, _I, _P, _P, _P, _P, _P, _P, C.c_int64, C.c_int64, _I, _D, C.c_int64, _P, _LL,
                         _P, _P], C.c_int),
    "ms_policy_max_jobs": ([_I], C.c_int),
    "ms_last_error": ([], C.c_char_p),
    "ms_device_sync": ([], C.c_int),
    "ms_policy_select": ([_P, _P, _P, _I, _P, C.c_int64, _D, _I, _P, _P], C.c_int),
    "ms_compact_index": ([_P, _I, _I, _P, _P, _P, _P, _P, _P], C.c_int),
    "ms_gather_rows": ([_P, _LL, _P, _P, _P, _I, _P, _P], C.c_int),
    "ms_gather_rows_pad": ([_P, _LL, _I, _I, _I, _I, _P, _P, _P, _I, _P, _P], C.c_int),
    "ms_compact": ([_P, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P], C.c_int),
    "ms_compact_ring": ([_P, _I, _I, _P, _P, _P, _I, _P, _P, _P, _P, _P, _P, _P], C.c_int),
    "ms_pass_select": ([_I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, C.c_int64, _P, _P, _P, _P,
                        _LL, _P, _P], C.c_int),
    "ms_gemm_plan_dense": ([_P, _P, _I, _I, _LL, _P, _I, _I, _I, _P, _I, _I, _P, _LL, _I, _I, _P],
                           C.c_int),
    "ms_gemm_plan_conv": ([_P, _P, _I, _I, _I, _I, _LL, _I, _I, _I, _I, _P, _I, _I, _P, _I, _P, _LL,
                           _I, _I, _P, _I, _I, _I], C.c_int),
    "ms_gemm_plan_conv_k32": ([_P, _P, _I, _I, _I, _I, _LL, _I, _I, _I, _I, _P, _I, _I, _P, _I, _P, _LL,
                               _I, _I, _P, _I, _I, _I], C.c_int),
    "ms_gemm_plan_conv_halo": ([_P, _P, _I, _I, _I, _I, _LL, _P, _I, _I, _P, _I, _P, _LL, _I, _I, _P], C.c_int),
    "ms_gemm_plan_stem_pool": ([_P, _P, _I, _I, _I, _I, _I, _I, _LL, _P, _P, _P, _LL, _I], C.c_int),
    "ms_gemm_plan_conv_pool": ([_P, _P, _I, _I, _I, _I, _LL, _P, _I, _P, _P, _LL, _I], C.c_int),
    "ms_gemm_plan_stem_set_reduce": ([_P, _P, _P, _P, _LL, _I], C.c_int),
    "ms_stream_wait_event": ([_P, _P], C.c_int),
    "ms_graph_launch": ([_P, _P], C.c_int),
    "ms_gemm_plan_gather": ([_P, _P, _P, _I, _I, _I, _I, _P, _I, _I, _P, _I, _I, _P, _LL, _I],
                            C.c_int),
    "ms_gemm_plan_fused_head": ([_P, _P, _P, _I, _I, _I, _I, _P, _P, _P, _P, _I, _P, _LL], C.c_int),
    "ms_gemm_plan_head_gemv": ([_P, _P, _P, _I, _I, _I, _I, _P, _P, _P, _P, _I, _P, _LL, _P, _P], C.c_int),
    "ms_gemm_run": ([_P, _P], C.c_int),
    "ms_gemm_plan_info": ([_P, _P, _P, _P, _P], C.c_int),
    "ms_pool2d": ([_P, _I, _I, _I, _I, _LL, _I, _I, _I, _I, _I, _P, _LL, _I, _P], C.c_int),
    "ms_pool2d_ex": ([_P, _I, _I, _I, _I, _LL, _I, _I, _I, _I, _I, _P, _LL, _I, _P, _I, _P], C.c_int),
    "ms_op_pool2d_ex": ([_P, _P, _I, _I, _I, _I, _LL, _I, _I, _I, _I, _I, _P, _LL, _I, _P, _I],
                        C.c_int),
    "ms_im2col": ([_P, _I, _I, _I, _I, _I, _I, _I, _I, _P, _I, _P], C.c_int),
    "ms_segment_mean": ([_P, _I, _I, _I, _I, _P, _LL, _P], C.c_int),
    "ms_op_gemm": ([_P, _P], C.c_int),
    "ms_op_pool2d": ([_P, _P, _I, _I, _I, _I, _LL, _I, _I, _I, _I, _I, _P, _LL, _I], C.c_int),
    "ms_op_im2col": ([_P, _P, _I, _I, _I, _I, _I, _I, _I, _I, _P, _I], C.c_int),
    "ms_op_segment_mean": ([_P, _P, _I, _I, _I, _I, _P, _LL], C.c_int),
    "ms_program_run": ([_P, _I, _P], C.c_int),
    "ms_event_create": ([_P], C.c_int),
    "ms_event_destroy": ([_P], C.c_int),
    "ms_event_record": ([_P, _P], C.c_int),
    "ms_event_elapsed_us": ([_P, _P, _P], C.c_int),
    "ms_event_query": ([_P], C.c_int),
    "ms_gemm_plan_set_residual": ([_P, _P, _LL], C.c_int),
    "ms_gemm_plan_set_splitk": ([_P, _I, _P, _LL], C.c_int),
    "ms_gemm_plan_debug": ([_P, _I], C.c_int),
    "ms_gemm_plan_set_trace": ([_P, _P], C.c_int),
    "ms_gemm_plan_set_pair": ([_P, _I], C.c_int),
    "ms_layernorm": ([_P, _LL, _LL, _P, _P, _P, _LL, _I, C.c_float, _P], C.c_int),
    "ms_attention": ([_P, _LL, _I, _I, _I, _P, _LL, C.c_float, _P], C.c_int),
    "ms_patchify": ([_P, _I, _I, _I, _I, _P, _P], C.c_int),
    "ms_vit_embed": ([_P, _P, _P, _I, _I, _I, _P, _P], C.c_int),
    "ms_bert_embed": ([_P, _LL, _I, _P, _P, _P, _P, _P, _P, _I, C.c_float, _P], C.c_int),
    "ms_op_layernorm": ([_P, _P, _LL, _LL, _P, _P, _P, _LL, _I, C.c_float], C.c_int),
    "ms_op_attention": ([_P, _P, _LL, _I, _I, _I, _P, _LL, C.c_float], C.c_int),
    "ms_op_patchify": ([_P, _P, _I, _I, _I, _I, _P], C.c_int),
    "ms_op_vit_embed": ([_P, _P, _P, _P, _I, _I, _I, _P], C.c_int),
    "ms_op_bert_embed": ([_P, _P, _LL, _I, _P, _P, _P, _P, _P, _P, _I, C.c_float], C.c_int),
}
EXPORTS = tuple(_SIGS)


def lib():
    """Load (once) and return the library; raises if it was not built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} missing: run `python -m paper_2310_18481_b200.build`")
        h = C.CDLL(str(LIB_PATH))
        for name, (args, res) in _SIGS.items():
            fn = getattr(h, name)
            fn.argtypes = args
            fn.restype = res
        _lib = h
    return _lib


def set_pdl(enable: bool) -> bool:
    """Programmatic dependent launch for op-program kernels (default on);
    returns the previous setting.  Affects plans launched afterwards."""
    return bool(lib().ms_set_pdl(int(bool(enable))))


def set_occ2_grid(mode: int) -> int:
    """Grid policy of two-CTAs-per-SM GEMM plans built afterwards (see
    ms_set_occ2_grid); returns the previous setting."""
    return int(lib().ms_set_occ2_grid(int(mode)))


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = lib().ms_last_error().decode(errors="replace")
        raise DeviceError(f"{what}: {msg} (status {rc})")


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("the B200 hot path needs a CUDA device; there is no CPU fallback")
    return torch


def stream_ptr(stream=None) -> int:
    """Raw cudaStream_t of ``stream`` (default: the current stream, read through
    the C binding: torch.cuda.current_stream() costs ~14 us of Python per call,
    which the serving loop pays several times per pass)."""
    if stream is not None:
        return stream.cuda_stream
    torch = _torch()
    return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())


def stream_wait(stream_p: int, ev: "Event") -> None:
    check(lib().ms_stream_wait_event(stream_p, ev.h), "ms_stream_wait_event")


def graph_launch(graph_exec: int, stream_p: int) -> None:
    check(lib().ms_graph_launch(graph_exec, stream_p), "ms_graph_launch")


def ptr(t) -> int | None:
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    return t.data_ptr()


def sync() -> None:
    check(lib().ms_device_sync(), "ms_device_sync")


# ------------------------------------------------------------------ policy


def policy_select(lat_us, credit, n_cand, deadline_us, dispatch_us: int, factor: float,
                  device=None, out=None, stream=None):
    """Device P5 over an SoA table. Accepts numpy or torch inputs; returns a
    numpy int32 array (or fills the CUDA tensor ``out`` without syncing)."""
    torch = _torch()
    dev = device or torch.device("cuda")

    def as_dev(a, dt):
        if isinstance(a, torch.Tensor):
            return a.to(device=dev, dtype=dt).contiguous()
        return torch.as_tensor(np.ascontiguousarray(a)).to(device=dev, dtype=dt)

    lat = as_dev(lat_us, torch.int64)
    n = lat.shape[0]
    cand = as_dev(n_cand, torch.int32)
    dl = as_dev(deadline_us, torch.int64)
    cr = as_dev(credit, torch.int32) if credit is not None else None
    res = out if out is not None else torch.empty(n, dtype=torch.int32, device=dev)
    check(lib().ms_policy_select(ptr(lat), ptr(cr), ptr(cand), int(lat.shape[1]), ptr(dl),
                                 int(dispatch_us), float(factor), int(n), ptr(res),
                                 stream_ptr(stream)), "ms_policy_select")
    if out is not None:
        return out
    return res.cpu().numpy()


def pass_select(n_prob, prob_job_off, prob_n_jobs, prob_now_us, prob_factor, job_size, job_deadline_us,
                job_n_cand, job_cand_off, job_mask_off, cand_counts, req_masks, cost: PassCost, cap: int,
                max_pass_ns: int, out_choice, out_summary, out_est_ns, out_mask, out_mask_ld: int, stream=None,
                out_clock=None):
    """ms_pass_select on raw addresses (device or pinned host memory): every
    array argument is an integer address (``tensor.data_ptr()``)."""
    check(lib().ms_pass_select(int(n_prob), prob_job_off, prob_n_jobs, prob_now_us, prob_factor, job_size,
                               job_deadline_us, job_n_cand, job_cand_off, job_mask_off, cand_counts, req_masks,
                               C.byref(cost), int(cap), int(max_pass_ns), out_choice, out_summary, out_est_ns,
                               out_mask, int(out_mask_ld), out_clock, stream_ptr(stream)), "ms_pass_select")


# -------------------------------------------------------------- compaction


def compact_index(mask, n_modalities: int, stream=None):
    """Device G1/G2 index build. ``mask`` is a CUDA uint16/int tensor [N].
    Returns (idx[K,N], inv[K,N], counts[K], combo_offsets[2^K+1], perm[N])."""
    torch = _torch()
    m = mask.to(torch.int16).contiguous() if mask.dtype != torch.int16 else mask.contiguous()
    n = m.shape[0]
    k = n_modalities
    dev = m.device
    idx = torch.full((k, max(n, 1)), -1, dtype=torch.int32, device=dev)
    inv = torch.empty((k, max(n, 1)), dtype=torch.int32, device=dev)
    counts = torch.empty(k, dtype=torch.int32, device=dev)
    offs = torch.empty((1 << k) + 1, dtype=torch.int32, device=dev)
    perm = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    check(lib().ms_compact_index(ptr(m), n, k, ptr(idx), ptr(inv), ptr(counts), ptr(offs),
                                 ptr(perm), stream_ptr(stream)), "ms_compact_index")
    return idx[:, :n], inv[:, :n], counts, offs, perm[:n]


def gather_rows(src, idx, count, max_rows: int, dst, slot=None, stream=None):
    row_bytes = src[0].numel() * src.element_size() if src.dim() > 1 else src.element_size()
    check(lib().ms_gather_rows(ptr(src), row_bytes, ptr(slot), ptr(idx), ptr(count), int(max_rows),
                               ptr(dst), stream_ptr(stream)), "ms_gather_rows")
    return dst


# ------------------------------------------------------------------ GEMMs


class GemmPlan:
    """An opaque 64-byte-aligned plan blob plus the tensors it points at
    (kept alive for the plan's lifetime)."""

    def __init__(self):
        self._raw = C.create_string_buffer(GEMM_PLAN_BYTES + 64)
        addr = C.addressof(self._raw)
        self.addr = (addr + 63) & ~63
        self.keep = []
        self.flops = 0
        self.label = ""
        self.split_k = 1

    def run(self, stream=None):
        check(lib().ms_gemm_run(self.addr, stream_ptr(stream)), "ms_gemm_run")

    def set_pair(self, enable: bool = True):
        """Run as 2-CTA clusters (tcgen05.mma.cta_group::2, M=256 tiles)."""
        check(lib().ms_gemm_plan_set_pair(self.addr, int(enable)), "ms_gemm_plan_set_pair")
        self.pair = bool(enable)
        return self

    def info(self):
        vals = [C.c_int() for _ in range(4)]
        check(lib().ms_gemm_plan_info(self.addr, *[C.byref(v) for v in vals]), "ms_gemm_plan_info")
        return {k: v.value for k, v in zip(("grid_x", "grid_y", "stages", "smem_bytes"), vals)}


def _segments(segs):
    if not segs:
        return 0, None
    arr = (Segment * len(segs))()
    for i, sg in enumerate(segs):
        nb, ne, t, ldd, col0 = sg[:5]
        arr[i] = Segment(nb, ne, ptr(t), ldd, col0, sg[5] if len(sg) > 5 else 0)
    return len(segs), arr


ACT_NONE, ACT_RELU, ACT_GELU, ACT_TANH = 0, 1, 2, 3


SM_COUNT = 148


def _auto_splitk(p, M, N, BN, num_kb, split_k, dev):
    """Split K when the output tiles cannot fill the GPU and K is deep:
    ksplit ~ SMs / tiles, each part >= 4 K blocks."""
    import torch
    tiles = -(-M // 128) * -(-N // BN)
    if split_k is None:
        # memset + finalize cost ~2 launches: only worth it for deep K on
        # a grid that leaves most SMs idle
        split_k = 1
        if tiles * 4 <= SM_COUNT and num_kb >= 16:
            split_k = max(1, min(num_kb // 4, SM_COUNT // tiles))
    if split_k > 1:
        ws_ld = -(-N // 4) * 4
        # one [M, ws_ld] fp32 slab per K part (summed in order by the finalize)
        ws = torch.empty(split_k * M, ws_ld, dtype=torch.float32, device=dev)
        check(lib().ms_gemm_plan_set_splitk(p.addr, split_k, ws.data_ptr(), ws_ld), "ms_gemm_plan_set_splitk")
        p.keep.append(ws)
        p.split_k = split_k
    return p


def _auto_pair(p, n_m_tiles, BN, allowed, N=0):
    """Use 2-SM CTA pairs where they measured faster (tools/gemm_bench.py,
    tools/pair_sweep.py): wide tiles (BN >= 128) with at least two waves of
    256-row tiles, or one wave of 128-row tiles with N >= 2048 (the ViT/BERT
    QKV and FC1 GEMMs: 1.02-1.06x)."""
    if allowed and BN >= 128 and getattr(p, "split_k", 1) == 1 and \
            (n_m_tiles >= 4 * SM_COUNT or (n_m_tiles >= SM_COUNT and N >= 2048)):
        p.set_pair()
    return p


def plan_dense(A, W, bias, D, *, K=None, BN=128, relu=False, out_fp32=False, col0=0, ldd=None,
               segs=None, M=None, act=None, residual=None, lda=None, split_k=None, pair=None):
    """D = act(A[M,K] @ W[N,K_pad]^T + bias) (+ residual); A row stride =
    ``lda`` or A.stride(0).  ``act`` is ACT_* (``relu=True`` == ACT_RELU)."""
    p = GemmPlan()
    m = A.shape[0] if M is None else M
    k = A.shape[1] if K is None else K
    nseg, sarr = _segments(segs)
    a = int(relu) if act is None else int(act)
    check(lib().ms_gemm_plan_dense(p.addr, ptr(A), m, k, A.stride(0) if lda is None else lda, ptr(W),
                                   W.shape[0], W.shape[1], BN, ptr(bias), a, int(out_fp32), ptr(D),
                                   D.stride(0) if ldd is None else ldd, col0, nseg, sarr),
          "ms_gemm_plan_dense")
    if residual is not None:
        check(lib().ms_gemm_plan_set_residual(p.addr, ptr(residual), residual.stride(0)),
              "ms_gemm_plan_set_residual")
    p.keep = [A, W, bias, D, segs, residual]
    p.flops = 2 * m * W.shape[0] * k
    p.label = f"dense M={m} N={W.shape[0]} K={k}"
    if not segs or len(segs) == 1:
        _auto_splitk(p, m, W.shape[0], BN, W.shape[1] // 64, split_k, A.device)
    if pair is not False and not out_fp32 and residual is None:
        if pair:
            p.set_pair()
        else:
            _auto_pair(p, -(-m // 128), BN, True, W.shape[0])
    return p


def plan_conv(X, n_img, H, W_in, C_in, c_stride, KH, KW, stride, pad, Wt, Cout, bias, D, *, ldd,
              col0=0, BN=128, relu=True, segs=None, tile=(1, 8, 16), pair=None, split_k=None, halo=False,
              k32=False):
    """Implicit-GEMM conv plan.  ``halo=True`` (3x3/1/1, width 14..62, >= 64
    channels): one halo box per channel chunk, taps as shifted smem views.
    ``k32=True`` (3x3, channels a multiple of 32 but not 64): K = 9*C exactly;
    ``Wt`` then comes from ``encoders.pack_conv_weight_k32``."""
    if k32:
        p = GemmPlan()
        nseg, sarr = _segments(segs)
        bn, bh, bw = tile
        check(lib().ms_gemm_plan_conv_k32(p.addr, ptr(X), n_img, H, W_in, C_in, c_stride, KH, KW, stride, pad,
                                          ptr(Wt), Cout, BN, ptr(bias), int(relu), ptr(D), ldd, col0, nseg, sarr,
                                          bn, bh, bw), "ms_gemm_plan_conv_k32")
        p.keep = [X, Wt, bias, D, segs]
        oh = (H + 2 * pad - KH) // stride + 1
        ow = (W_in + 2 * pad - KW) // stride + 1
        p.flops = 2 * n_img * oh * ow * Cout * KH * KW * C_in
        p.label = f"conv {KH}x{KW}/{stride} {C_in}->{Cout} {n_img}x{oh}x{ow} k32"
        return p
    if halo:
        p = GemmPlan()
        nseg, sarr = _segments(segs)
        check(lib().ms_gemm_plan_conv_halo(p.addr, ptr(X), n_img, H, W_in, C_in, c_stride, ptr(Wt), Cout, BN,
                                           ptr(bias), int(relu), ptr(D), ldd, col0, nseg, sarr),
              "ms_gemm_plan_conv_halo")
        p.keep = [X, Wt, bias, D, segs]
        p.flops = 2 * n_img * H * W_in * Cout * 9 * C_in
        p.label = f"conv 3x3/1 {C_in}->{Cout} {n_img}x{H}x{W_in} halo"
        return p
    p = GemmPlan()
    nseg, sarr = _segments(segs)
    bn, bh, bw = tile
    check(lib().ms_gemm_plan_conv(p.addr, ptr(X), n_img, H, W_in, C_in, c_stride, KH, KW, stride, pad,
                                  ptr(Wt), Cout, BN, ptr(bias), int(relu), ptr(D), ldd, col0, nseg,
                                  sarr, bn, bh, bw), "ms_gemm_plan_conv")
    p.keep = [X, Wt, bias, D, segs]
    oh = (H + 2 * pad - KH) // stride + 1
    ow = (W_in + 2 * pad - KW) // stride + 1
    p.flops = 2 * n_img * oh * ow * Cout * KH * KW * C_in
    p.label = f"conv {KH}x{KW}/{stride} {C_in}->{Cout} {n_img}x{oh}x{ow}"
    bn_, bh_, bw_ = tile
    conv_tiles = -(-n_img // bn_) * -(-oh // bh_) * -(-ow // bw_)
    if C_in >= 64 and (not segs or len(segs) == 1) and split_k is not None and split_k > 1:
        # explicit only: splitting the (tap, channel-chunk) K loop of the small
        # late layers measured SLOWER inside a pass (fp32 atomics + finalize
        # outweigh the idle SMs it fills; tools/pass_ab.py, round 1)
        k = split_k
        if k > 1:
            m_rows = n_img * oh * ow
            ws_ld = -(-Cout // 4) * 4
            ws = _torch().empty(k * m_rows, ws_ld, dtype=_torch().float32, device=D.device)
            check(lib().ms_gemm_plan_set_splitk(p.addr, k, ws.data_ptr(), ws_ld), "ms_gemm_plan_set_splitk")
            p.keep.append(ws)
            p.split_k = k
            return p
    if C_in >= 64 and pair is not False:  # not the small-channel first layer
        if pair:
            p.set_pair()
        else:
            bn_, bh_, bw_ = tile
            _auto_pair(p, conv_tiles, BN, True)
    return p


def plan_stem_pool(X, n_img, H, W_in, KH, pad, Wt, bias, Y, *, ldy, col0=0, planes=1, plane_stride=0):
    """Fused 7x7/2 conv (4-channel pre-padded pixels, or three 4-channel
    planes, 64 out, ReLU) + 3x3/2 ceil max pool (``ms_gemm_plan_stem_pool``);
    ``Wt`` from ``encoders.pack_stem_weight`` (``_planes`` for 3 planes)."""
    p = GemmPlan()
    check(lib().ms_gemm_plan_stem_pool(p.addr, ptr(X), n_img, H, W_in, KH, pad, planes, plane_stride, ptr(Wt),
                                       ptr(bias), ptr(Y), ldy, col0), "ms_gemm_plan_stem_pool")
    p.keep = [X, Wt, bias, Y]
    oh = (H + 2 * pad - KH) // 2 + 1
    ow = (W_in + 2 * pad - KH) // 2 + 1
    p.flops = 2 * n_img * oh * ow * 64 * KH * KH * 4 * planes
    p.label = f"stem conv {KH}x{KH}/2 {4 * planes}->64 {n_img}x{oh}x{ow} + maxpool"
    return p


def stem_set_reduce(p, Wred, bias, Y, *, ldy, col0=0):
    """Fuse the 64 -> 64 1x1 conv (+ bias + ReLU) into stem plan ``p``
    (``ms_gemm_plan_stem_set_reduce``); ``Wred`` from
    ``encoders.pack_sw128_weight``.  The plan then writes Y instead of the
    pooled map."""
    check(lib().ms_gemm_plan_stem_set_reduce(p.addr, ptr(Wred), ptr(bias), ptr(Y), ldy, col0),
          "ms_gemm_plan_stem_set_reduce")
    p.keep += [Wred, bias, Y]
    p.label += " + 1x1 64->64"
    return p


def plan_conv_pool(X, n_img, H, W_in, C_in, c_stride, Wt, Cout, bias, Y, *, ldy, col0=0):
    """Fused 3x3/1/1 conv + bias + ReLU + 3x3/2 ceil max pool
    (``ms_gemm_plan_conv_pool``, widths 55..62 or 64): the pooled map is written to
    ``Y`` ([n_img, PH, PW] rows of ``ldy``), the conv map never reaches HBM.
    ``Wt`` from ``encoders.pack_conv_weight``."""
    p = GemmPlan()
    check(lib().ms_gemm_plan_conv_pool(p.addr, ptr(X), n_img, H, W_in, C_in, c_stride, ptr(Wt), Cout, ptr(bias),
                                       ptr(Y), ldy, col0), "ms_gemm_plan_conv_pool")
    p.keep = [X, Wt, bias, Y]
    p.flops = 2 * n_img * H * W_in * Cout * 9 * C_in
    p.label = f"conv_pool_kernel conv 3x3/1 {C_in}->{Cout} {n_img}x{H}x{W_in} + maxpool 3x3/2"
    return p


def plan_gather(feats, inv, W, bias, D, *, M, feat_dim, BN=128, relu=True, out_fp32=False,
                split_k=None):
    p = GemmPlan()
    arr = (C.c_void_p * len(feats))(*[ptr(f) for f in feats])
    check(lib().ms_gemm_plan_gather(p.addr, arr, ptr(inv), inv.stride(0), len(feats), feat_dim, M,
                                    ptr(W), W.shape[0], BN, ptr(bias), int(relu), int(out_fp32),
                                    ptr(D), D.stride(0), 0), "ms_gemm_plan_gather")
    p.keep = [feats, inv, W, bias, D, arr]
    p.flops = 2 * M * W.shape[0] * len(feats) * feat_dim
    p.label = f"gather-concat M={M} N={W.shape[0]} K={len(feats) * feat_dim}"
    _auto_splitk(p, M, W.shape[0], BN, len(feats) * feat_dim // 64, split_k, W.device)
    return p


def plan_fused_head(feats, inv, W1, b1, W2, b2, logits, *, M, feat_dim):
    """The late-fusion head in one cluster launch (ms_gemm_plan_fused_head):
    gather-concat FC1 + ReLU + FC2 -> fp32 logits[:M]."""
    p = GemmPlan()
    arr = (C.c_void_p * len(feats))(*[ptr(f) for f in feats])
    check(lib().ms_gemm_plan_fused_head(p.addr, arr, ptr(inv), inv.stride(0), len(feats), feat_dim, M, ptr(W1),
                                        ptr(b1), ptr(W2), ptr(b2), W2.shape[0], ptr(logits), logits.stride(0)),
          "ms_gemm_plan_fused_head")
    p.keep = [feats, inv, W1, b1, W2, b2, logits, arr]
    p.flops = 2 * M * W1.shape[0] * len(feats) * feat_dim + 2 * M * W1.shape[0] * W2.shape[0]
    p.label = f"fused_head_kernel M={M} K={len(feats) * feat_dim} -> {W1.shape[0]} -> {W2.shape[0]}"
    return p


def plan_head_gemv(feats, inv, W1, b1, W2, b2, logits, h, *, M, feat_dim):
    """The late-fusion head for small passes (ms_gemm_plan_head_gemv): FC1 as
    a weight stream over 128 CTAs -> bf16 h -> grid barrier -> FC2, one launch."""
    import torch
    p = GemmPlan()
    sync = torch.zeros(2, dtype=torch.int32, device=W1.device)  # barrier count + generation
    arr = (C.c_void_p * len(feats))(*[ptr(f) for f in feats])
    check(lib().ms_gemm_plan_head_gemv(p.addr, arr, ptr(inv), inv.stride(0), len(feats), feat_dim, M, ptr(W1),
                                       ptr(b1), ptr(W2), ptr(b2), W2.shape[0], ptr(logits), logits.stride(0),
                                       ptr(h), ptr(sync)), "ms_gemm_plan_head_gemv")
    p.keep = [feats, inv, W1, b1, W2, b2, logits, h, sync, arr]
    p.flops = 2 * M * W1.shape[0] * len(feats) * feat_dim + 2 * M * W1.shape[0] * W2.shape[0]
    p.label = f"head_gemv_kernel M={M} K={len(feats) * feat_dim} -> {W1.shape[0]} -> {W2.shape[0]}"
    return p


# -------------------------------------------------------------- op programs


class Program:
    """A native op list (ms_program_run): one call runs a whole encoder."""

    def __init__(self):
        self.ops = []  # (kind, args)
        self.keep = []
        self._buf = None
        self._addr = 0

    def gemm(self, plan: GemmPlan):
        self.ops.append(("gemm", plan))
        self.keep.append(plan)

    def pool(self, X, n_img, H, W, C_, x_cs, k, stride, pad, ceil_mode, is_max, Y, y_cs, y_col0,
             bias=None, relu=False):
        self.ops.append(("pool", (ptr(X), n_img, H, W, C_, x_cs, k, stride, pad, int(ceil_mode),
                                  int(is_max), ptr(Y), y_cs, y_col0, ptr(bias), int(relu))))
        self.keep += [X, Y, bias]

    def im2col(self, X, n_img, H, W, C_, KH, KW, stride, pad, out, K_pad):
        self.ops.append(("im2col", (ptr(X), n_img, H, W, C_, KH, KW, stride, pad, ptr(out), K_pad)))
        self.keep += [X, out]

    def segment_mean(self, X, n_req, S, HW, C_, Y, y_ld):
        self.ops.append(("segmean", (ptr(X), n_req, S, HW, C_, ptr(Y), y_ld)))
        self.keep += [X, Y]

    def layernorm(self, X, ldx, rows, gamma, beta, Y, ldy, C_, eps=1e-6):
        self.ops.append(("ms_op_layernorm", (ptr(X), ldx, rows, ptr(gamma), ptr(beta), ptr(Y), ldy, C_,
                                             float(eps))))
        self.keep += [X, gamma, beta, Y]

    def attention(self, qkv, ld, L, H, n_seq, out, ldo, scale):
        self.ops.append(("ms_op_attention", (ptr(qkv), ld, L, H, n_seq, ptr(out), ldo, float(scale))))
        self.keep += [qkv, out]

    def patchify(self, X, n, S, C_, P_, Y):
        self.ops.append(("ms_op_patchify", (ptr(X), n, S, C_, P_, ptr(Y))))
        self.keep += [X, Y]

    def vit_embed(self, pe, cls, pos, n, L, D, tok):
        self.ops.append(("ms_op_vit_embed", (ptr(pe), ptr(cls), ptr(pos), n, L, D, ptr(tok))))
        self.keep += [pe, cls, pos, tok]

    def bert_embed(self, ids, n_tok, L, word, pos, type0, gamma, beta, Y, D, eps=1e-12):
        self.ops.append(("ms_op_bert_embed", (ptr(ids), n_tok, L, ptr(word), ptr(pos), ptr(type0),
                                              ptr(gamma), ptr(beta), ptr(Y), D, float(eps))))
        self.keep += [ids, word, pos, type0, gamma, beta, Y]

    def seal(self):
        n = len(self.ops)
        self._buf = C.create_string_buffer(OP_BYTES * max(n, 1) + 64)
        self._addr = (C.addressof(self._buf) + 63) & ~63
        L = lib()
        for i, (kind, a) in enumerate(self.ops):
            at = self._addr + i * OP_BYTES
            if kind == "gemm":
                check(L.ms_op_gemm(at, a.addr), "ms_op_gemm")
            elif kind == "pool":
                check(L.ms_op_pool2d_ex(at, *a), "ms_op_pool2d_ex")
            elif kind == "im2col":
                check(L.ms_op_im2col(at, *a), "ms_op_im2col")
            elif kind == "segmean":
                check(L.ms_op_segment_mean(at, *a), "ms_op_segment_mean")
            else:
                check(getattr(L, kind)(at, *a), kind)
        return self

    def run(self, stream=None):
        if self._buf is None:
            self.seal()
        check(lib().ms_program_run(self._addr, len(self.ops), stream_ptr(stream)), "ms_program_run")

    @property
    def n_launches(self) -> int:
        # a split-K GEMM is two launches (tiles + finalize)
        return sum(2 if k == "gemm" and getattr(a, "split_k", 1) > 1 else 1 for k, a in self.ops)


class StagedProgram:
    """Native programs arranged as a sequence of stages; a stage's lanes are
    independent (e.g. the branches of an Inception block) and run
    concurrently on side streams, forked from and joined back into the
    calling stream.  Captured in a CUDA graph this is a DAG, so small-batch
    branches fill SMs the trunk leaves idle.  ``streams``/``events`` are
    shared by every program of one encoder (its programs never overlap)."""

    def __init__(self, lanes_ctx):
        self.stages = []  # list[list[Program]]
        self.ctx = lanes_ctx

    def stage(self, *lanes):
        lanes = [p for p in lanes if p is not None and p.ops]
        if lanes:
            self.stages.append(lanes)
        return self

    def seal(self):
        for lanes in self.stages:
            for p in lanes:
                p.seal()
        return self

    @property
    def ops(self):
        return [op for lanes in self.stages for p in lanes for op in p.ops]

    @property
    def keep(self):
        return [k for lanes in self.stages for p in lanes for k in p.keep]

    @property
    def n_launches(self) -> int:
        return sum(p.n_launches for lanes in self.stages for p in lanes)

    def first(self):
        """Stage 0 alone (a StagedProgram view sharing the sealed programs)."""
        v = StagedProgram(self.ctx)
        v.stages = self.stages[:1]
        return v

    def tail(self):
        """Every stage after stage 0 (a StagedProgram view)."""
        v = StagedProgram(self.ctx)
        v.stages = self.stages[1:]
        return v

    def run(self, stream=None):
        torch = _torch()
        main = torch.cuda.current_stream() if stream is None else stream
        side, ev_fork, ev_join = self.ctx.streams, self.ctx.fork, self.ctx.join
        for lanes in self.stages:
            if len(lanes) == 1 or not self.ctx.concurrent:
                for p in lanes:
                    p.run(main)
                continue
            ev_fork.record(main)
            for i, p in enumerate(lanes[1:]):
                side[i].wait_event(ev_fork)
                p.run(side[i])
                ev_join[i].record(side[i])
            lanes[0].run(main)
            for i in range(len(lanes) - 1):
                main.wait_event(ev_join[i])


class LaneContext:
    """Side streams + fork/join events for StagedProgram lanes."""

    def __init__(self, n_side: int = 2, concurrent: bool = True):
        torch = _torch()
        self.concurrent = concurrent  # False: lanes run one after another (A/B)
        self.streams = [torch.cuda.Stream() for _ in range(n_side)]
        self.fork = torch.cuda.Event()
        self.join = [torch.cuda.Event() for _ in range(n_side)]


# ------------------------------------------------------------------ events


class Event:
    def __init__(self):
        h = C.c_void_p()
        check(lib().ms_event_create(C.byref(h)), "ms_event_create")
        self.h = h

    def record(self, stream=None):
        check(lib().ms_event_record(self.h, stream_ptr(stream)), "ms_event_record")

    def record_on(self, stream_p: int):
        """Record on a raw cudaStream_t (no stream object lookup)."""
        check(lib().ms_event_record(self.h, stream_p), "ms_event_record")

    def done(self) -> bool:
        """True once the device has passed this event (non-blocking)."""
        rc = lib().ms_event_query(self.h)
        if rc < 0:
            check(MS_ERR_CUDA_STATUS, "ms_event_query")
        return rc == 0

    def elapsed_us(self, end: "Event") -> float:
        out = C.c_double()
        check(lib().ms_event_elapsed_us(self.h, end.h, C.byref(out)), "ms_event_elapsed_us")
        return out.value

    def __del__(self):
        try:
            if _lib is not None and self.h:
                _lib.ms_event_destroy(self.h)
        except Exception:
            pass
