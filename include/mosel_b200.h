/* mosel_b200.h — C-ABI of the B200 (sm_100a) hot path of MOSEL-style
 * modality-aware serving (arXiv 2310.18481; reference package `modserve`).
 *
 * The reference is pure Python and has no FFI layer; its
 * worker seam is a table lookup.  Each entry point below replaces one
 * reference interface, cited file:line into /root/reference/pkg/src/modserve:
 *
 *   ms_policy_select  <- scheduler.py:382-425 apply_policy(OPTIMIZED) on a
 *                        one-job scope (+ :202-233 detect_violation /
 *                        compute_budget, :236-326 reassign_optimized,
 *                        :366-379 try_upgrade); closed form SURVEY §8a P5.
 *   ms_compact_index  <- strategy.py:54-60 Strategy.make canonical (mask,
 *   ms_gather_rows       batch) grouping + sim.py:372-377 part loop: turns
 *   ms_compact           per-request masks into modality-grouped sub-batches.
 *   ms_gemm_plan_*    <- sim.py:374 profile.part_latency_us(mask, batch)
 *   ms_gemm_run          stand-in: the per-modality encoders (dense layers,
 *   ms_op_* / ms_program_run   implicit-GEMM convolutions) and late fusion +
 *                        head; dropped modalities = all_mask & ~mask
 *                        (profile.py:157-159) contribute nothing.
 *   ms_event_* (profiler) <- profile.py:338-356 save_profile producer: the
 *                        latency table is refreshed from CUDA-event timings.
 *
 * Conventions: every call is stream-ordered on the `stream` argument
 * (a cudaStream_t passed as void*), takes caller-owned device pointers,
 * performs no allocation and returns an int status: 0 = MS_OK; nonzero maps
 * to the reference's ValueError family on the Python side; the message is
 * available from ms_last_error().  Plans/ops are caller-allocated opaque
 * blobs of MS_GEMM_PLAN_BYTES / MS_OP_BYTES bytes (64-byte aligned).
 */
#ifndef MOSEL_B200_H
#define MOSEL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define MS_OK 0
#define MS_ERR_INVALID 1
#define MS_ERR_CUDA 2

#define MS_GEMM_PLAN_BYTES 2048
#define MS_OP_BYTES 2112

#define MS_DROP (-1)

typedef struct MsSegment {
  int n_begin;   /* first output column of this segment */
  int n_end;     /* one past the last */
  void* ptr;     /* destination base */
  long long ldd; /* destination row stride (elements) */
  int col0;      /* destination column of n_begin */
  int flags;     /* MS_SEG_NO_RELU: store this segment pre-activation */
} MsSegment;
#define MS_SEG_NO_RELU 1

int ms_abi_version(void);
/* Programmatic dependent launch for op-program kernels (default on): the
 * next kernel's prologue overlaps the previous kernel's tail.  Returns the
 * previous setting. */
int ms_set_pdl(int enable);
/* Grid policy of the two-CTAs-per-SM GEMM plans built afterwards: 0 = one
 * CTA per SM, 1 = up to two (the kernel fills the GPU alone), 2 = two only
 * with >= 4 tiles per SM (leaves room for kernels running beside it), < 0 =
 * MS_OCC2_GRID / default 1.  Returns the previous setting. */
int ms_set_occ2_grid(int mode);
const char* ms_last_error(void);
int ms_device_sync(void);

/* ---- policy step (one warp per job) --------------------
 * lat_us[N*C] / credit[N*C]: per-job frontier (ascending latency, strictly
 * increasing credit), n_cand[N] valid entries, deadline_us[N];
 * est = round_half_even(lat * factor); B = deadline - dispatch_us.
 * choice[N] = index into the frontier or MS_DROP. credit may be NULL. */
int ms_policy_select(const int64_t* lat_us, const int32_t* credit, const int32_t* n_cand, int C,
                     const int64_t* deadline_us, int64_t dispatch_us, double factor, int N,
                     int32_t* choice, void* stream);

/* ---- pass-level selection (the batched executor's policy step) ---------
 * ms_pass_select <- the per-request argmax of scheduler.py:382-425 on a
 * one-job scope (ms_policy_select above) with the latency
 * budget coupled through ONE shared device pass: the batched executor's
 * policy step (SURVEY §8f #4 cross-job batching; the reference never
 * batches across jobs, and next_dispatch scheduler.py:428-449
 * still pops and drop-checks the head on the host).  One warp per problem:
 *   1. membership: the head + queued jobs in EDF order join at their fastest
 *      candidate while n <= cap, now + est <= every member's deadline and
 *      est <= max_pass_ns (< 0: none) -- warp prefix scans, first misfit ends;
 *   2. the jobs left queued: rest_fast = est(their fastest counts), rest_dl =
 *      earliest rest deadline >= now + est + rest_fast;
 *   3. each member in EDF order takes the LARGEST frontier index >= its
 *      current one whose pass estimate keeps every member, the rest and the
 *      cap on time (one warp ballot over its candidates), until none moves.
 * est(counts) = round_half_even(raw(sum_k w[k]*counts[k]) * factor) with raw
 * the integer piecewise-linear pass time of MsPassCost.  Restated bit-exactly
 * by oracle/selection.py pass_select.
 * Problem p: jobs prob_job_off[p] .. +prob_n_jobs[p] (index 0 = the head),
 * now (us) and EWMA factor.  Job j: size, deadline (us), n_cand frontier
 * entries whose per-modality request counts are cand_counts[(job_cand_off[j]
 * + c) * K + k] and whose per-request masks are req_masks[job_mask_off[j] +
 * c * size + i].  Outputs: out_choice[j] = chosen index for members, -1
 * otherwise; out_summary[p * MS_PASS_SUMMARY + ...] = {members, requests,
 * counts[K]}; out_est_ns[p]; out_mask[p * out_mask_ld + r] = the pass's
 * per-request masks (members in order).  Inputs/outputs may be device or
 * pinned (mapped) host memory: the serving loop hands the kernel its pinned
 * staging buffers directly (no memcpy), only out_mask lives in HBM.
 * out_clock (may be NULL): [2p], [2p+1] = the problem's start / end on the
 * device's global timer (ns) -- the kernel's own time, apart from queueing. */
#define MS_PASS_MAX_K 8
#define MS_PASS_MAX_PTS 32
#define MS_PASS_MAX_MEMBERS 1024
#define MS_PASS_SUMMARY (2 + MS_PASS_MAX_K)
typedef struct MsPassCost {
  int K, n_pts;
  int32_t w[MS_PASS_MAX_K];   /* work of one request's modality k, in 1/1024 all-modality requests */
  int64_t u[MS_PASS_MAX_PTS]; /* knots: work (same units), strictly increasing */
  int64_t t_ns[MS_PASS_MAX_PTS]; /* measured pass time at each knot (ns), non-decreasing */
} MsPassCost;
int ms_pass_select(int n_prob, const int32_t* prob_job_off, const int32_t* prob_n_jobs,
                   const int64_t* prob_now_us, const double* prob_factor, const int32_t* job_size,
                   const int64_t* job_deadline_us, const int32_t* job_n_cand, const int32_t* job_cand_off,
                   const int32_t* job_mask_off, const int16_t* cand_counts, const uint16_t* req_masks,
                   const MsPassCost* cost, int cap, int64_t max_pass_ns, int32_t* out_choice,
                   int32_t* out_summary, int64_t* out_est_ns, uint16_t* out_mask, long long out_mask_ld,
                   int64_t* out_clock, void* stream);

/* ms_strategy_dp <- strategy.py:139-177 _DpTables (offline stage, SURVEY
 * §8f #2): the exact min-latency / min-part-count table over (requests
 * covered r <= max_size, credit index c < max_size*unit+1) for items
 * (batch, latency_us, credit // gcd) in canonical order.  lat/cnt are device
 * arrays [max_size+1, max_size*unit+1]; unreachable = 2^62 / INT32_MAX, as in
 * the reference.  Query/back-walk stay on the host (byte-identical matrices). */
int ms_strategy_dp(int n_items, const int32_t* batch, const int64_t* lat_us, const int32_t* credit_idx, int max_size,
                   int unit, int64_t* lat, int32_t* cnt, void* stream);

/* ms_policy_apply <- scheduler.py:382-425 apply_policy(OPTIMIZED) over a whole
 * EDF queue (detect_violation -> compute_budget -> reassign_optimized MCKP,
 * scheduler.py:187-326 -> drops -> try_upgrade :366-379), one launch.
 * Jobs in EDF order; candidate tables [n, C] (lat_us, credit, effective
 * accuracy as double); assigned[n] in/out (-1 on return = dropped).
 * has_running: the running job's estimated finish sets the dispatch time
 * (scheduler.py:178-184).  grid_us = the knapsack quantum (reference 1000).
 * ws: device scratch of ws_bytes (16 bytes per knapsack cell; a queue never
 * needs more than (n + 1) * (floor((max deadline - dispatch) / grid_us) + 1)
 * cells); *status (device) = 0 ok, 1 scratch too small (a caller error).
 * n <= ms_policy_max_jobs(C) (per-job tables in shared memory).  Bit-exact
 * with the reference (tests/golden/queue_policy_cases.json). */
int ms_policy_apply(int n, int C, const int64_t* lat_us, const int32_t* credit, const double* acc,
                    const int32_t* n_cand, const int64_t* deadline_us, int32_t* assigned, int64_t now_us,
                    int64_t running_finish_us, int has_running, double factor, int64_t grid_us, void* ws,
                    long long ws_bytes, int32_t* status, void* stream);
/* the longest queue ms_policy_apply takes with C candidate columns (0 if C is out of range) */
int ms_policy_max_jobs(int C);

/* ---- request compaction ----------------------------
 * mask[N] (bit k = modality k present) ->
 *   idx[K*N]   : idx[k*N + j] = j-th request (ascending) that has modality k
 *   inv[K*N]   : inv[k*N + i] = position of request i in idx_k, or -1
 *   counts[K]  : |idx_k|
 *   combo_offsets[2^K + 1], perm[N]: stable counting sort of requests by mask */
int ms_compact_index(const uint16_t* mask, int N, int K, int32_t* idx, int32_t* inv, int32_t* counts,
                     int32_t* combo_offsets, int32_t* perm, void* stream);
/* dst[j] = src[slot ? slot[idx[j]] : idx[j]] for j < *count (count read on
 * device); rows of row_bytes (multiple of 16), vectorised 16-B copies. */
int ms_gather_rows(const void* src, long long row_bytes, const int32_t* slot, const int32_t* idx,
                   const int32_t* count, int max_rows, void* dst, void* stream);
/* One request row of a modality: `lines` lines of `width` pixels with c_src
 * channels in the pool; in the encoder input each pixel has c_dst (>= c_src,
 * multiple of 8) channels and every line gets pad_w zero pixels on both
 * ends (the first conv's window padding).  Plain rows: lines=1, width=1,
 * c_src=c_dst=elements, pad_w=0.  src_u8 pools are converted to bf16 on the
 * fly (halves host->device and HBM input bytes for video). */
typedef struct MsRowDesc {
  long long lines;
  int width, c_src, c_dst, pad_w; /* c_dst: 4 or a multiple of 8 */
  int src_u8;              /* 1: pool holds uint8 (frames, quantised flow) */
  float u8_scale, u8_bias; /* bf16 value = u8 * scale + bias */
  int frame_h, pad_h;      /* frames of frame_h lines get pad_h zero rows above/below (0: none) */
  int slot_off;            /* this modality's request->pool-row map is slot[slot_off + request] */
  long long plane_stride;  /* > 0 (c_dst == 12 only): write three 4-channel planes, plane q at
                              G + q * plane_stride elements (the fused stem's input layout) */
} MsRowDesc;
int ms_gather_rows_pad(const void* src, long long lines, int width, int c_src, int c_dst, int pad_w,
                       const int32_t* slot, const int32_t* idx, const int32_t* count, int max_rows,
                       void* dst, void* stream);
/* index + one gather per modality (K <= 8), rows described by rows[k] */
int ms_compact(const uint16_t* mask, int N, int K, const void* const* X, const MsRowDesc* rows,
               const int32_t* slot, void* const* G, int32_t* idx, int32_t* inv, int32_t* counts,
               int32_t* combo_offsets, int32_t* perm, void* stream);

/* as ms_compact, but modality k's compacted position j reads pool row
 * (ring_base[k] + j) % n_ring (ring_base: HOST array [K]) instead of a slot
 * map: the serving loop's per-modality input rings, where a pass's clips of
 * modality k occupy consecutive ring rows (one DMA per modality) */
int ms_compact_ring(const uint16_t* mask, int N, int K, const void* const* X, const MsRowDesc* rows,
                    const int32_t* ring_base, int n_ring, void* const* G, int32_t* idx, int32_t* inv,
                    int32_t* counts, int32_t* combo_offsets, int32_t* perm, void* stream);

/* ---- tcgen05 GEMM plans (encoders, fusion head) -----------------------
 * W is [N rows, K_pad] bf16 K-major (zero padded).  bias fp32[N] or NULL,
 * N <= 4096.  The `relu` argument is the epilogue activation MS_ACT_*. */
#define MS_ACT_NONE 0
#define MS_ACT_RELU 1
#define MS_ACT_GELU 2
#define MS_ACT_TANH 3
int ms_gemm_plan_dense(void* plan, const void* A, int M, int K, long long lda, const void* W, int N,
                       int K_pad, int BN, const float* bias, int relu, int out_fp32, void* D,
                       long long ldd, int col0, int nseg, const MsSegment* segs);
/* implicit-GEMM conv over NHWC bf16 input [n_img, H, W, C] (channel stride
 * c_stride); weights [Cout, KH*KW*ceil64(C)] tap-major, each tap's channels
 * zero-padded to a multiple of 64; output pixel-major [n_img*OH*OW, ...].
 * (bn, bh, bw) is the output-pixel block one 128-row tile covers.
 * C = 8 or 16: first-layer mode; X is [n_img, H, W_in + 2*pad, C] (W
 * pre-padded, e.g. by ms_compact's pad_w) and the weights are
 * [Cout, KH * 8 * C] in (kh, window pixel j < 8, c) order, taps j >= KW zero. */
int ms_gemm_plan_conv(void* plan, const void* X, int n_img, int H, int W_in, int C, long long c_stride,
                      int KH, int KW, int stride, int pad, const void* Wt, int Cout, int BN,
                      const float* bias, int relu, void* D, long long ldd, int col0, int nseg,
                      const MsSegment* segs, int bn, int bh, int bw);
/* masked late-fusion concat GEMM: row i, K slice k*F..(k+1)*F reads
 * feat[k][inv[k*inv_ld + i]] or zeros when inv == -1. */
/* 3x3 implicit-GEMM conv for input channels a multiple of 32 but not of 64:
 * K = 9 * C exactly, weights [Cout, ceil64(9*C)] in (tap, channel) order. */
int ms_gemm_plan_conv_k32(void* plan, const void* X, int n_img, int H, int W_in, int C, long long c_stride, int KH,
                          int KW, int stride, int pad, const void* Wt, int Cout, int BN, const float* bias, int relu,
                          void* D, long long ldd, int col0, int nseg, const MsSegment* segs, int bn, int bh, int bw);
/* 3x3 / stride 1 / pad 1 implicit-GEMM conv with halo reuse (widths 14..62,
 * >= 64 input channels): one TMA box of (bh+2) input rows x ceil8(W+2)
 * pixels per 64-channel chunk, the 9 taps read as shifted views of it;
 * otherwise as ms_gemm_plan_conv (same weights layout, outputs, segments). */
int ms_gemm_plan_conv_halo(void* plan, const void* X, int n_img, int H, int W_in, int C, long long c_stride,
                           const void* Wt, int Cout, int BN, const float* bias, int relu, void* D, long long ldd,
                           int col0, int nseg, const MsSegment* segs);
/* Fused stem: 7x7 (KH <= 8) / stride-2 conv over pre-padded 4-channel pixels
 * X [n_img, H + 2*pad, W + 2*pad, 4] bf16 (output width <= 128), 64 output
 * channels, + bias + ReLU, then the 3x3 / stride-2 / ceil-mode max pool, in
 * ONE kernel: Y = pooled [n_img, PH, PW] rows of ldy elements at y_col0.  The
 * input rows are the A operand as they lie (no-swizzle K-major descriptors
 * with overlapping core matrices); each input row feeds both conv rows of a
 * pair through N = 128 MMAs.  Wt: 9 x [128, 32] bf16 row-pair weights in the
 * no-swizzle core-matrix order (encoders.pack_stem_weight), 16-B aligned.
 * planes = 3 (flow, up to 12 channels): X holds three 4-channel planes
 * plane_stride elements apart (ms_compact's planar gather), N = 64 MMAs per
 * (conv row, filter row, plane), Wt = encoders.pack_stem_weight_planes. */
int ms_gemm_plan_stem_pool(void* plan, const void* X, int n_img, int H, int W_in, int KH, int pad, int planes,
                           long long plane_stride, const void* Wt, const float* bias, void* Y, long long ldy,
                           int y_col0);
/* Fused 3x3 / stride-1 / pad-1 conv + bias + ReLU + 3x3 / stride-2 ceil-mode
 * max pool (BN-Inception conv2 + pool2; reference consumer: the modality
 * encoder whose latency profile.py:96-212 tabulates).  X [n_img, H, W, C]
 * NHWC bf16 with 55 <= W <= 62 (halo rows of 64 pixels) or W == 64 (one
 * tap box per (chunk, tap)), and C >= 64 (pixel
 * stride c_stride), Wt [Cout, 9 * ceil64(C)] tap-major (encoders
 * .pack_conv_weight), Cout in {128, 192, 256}; Y = pooled [n_img, PH, PW]
 * rows of ldy elements at y_col0.  Bitwise equal to the halo conv followed
 * by ms_pool (same accumulation order); the unpooled map never reaches HBM. */
int ms_gemm_plan_conv_pool(void* plan, const void* X, int n_img, int H, int W_in, int C, long long c_stride,
                           const void* Wt, int Cout, const float* bias, void* Y, long long ldy, int y_col0);
/* The whole late-fusion head in one launch (replaces ms_gemm_plan_gather +
 * the FC2 dense plan + its split-K finalize; reference: the fusion MLP over
 * the concatenated encoder outputs, absent modalities zero -- profile.py:
 * 157-159).  logits[M, n_classes] (fp32, row stride ldo) = FC2(ReLU(FC1(
 * concat_k feat[k][inv[k, r]] or 0))): W1 [512, n_mod * feat_dim] bf16
 * K-major, b1 [512], W2 [n_classes, 512] bf16 K-major, b2 [n_classes].
 * Needs n_mod * feat_dim % 512 == 0 and n_classes <= 512.  8-CTA clusters per
 * 128 requests; FC1 and FC2 partials reduce-scatter over distributed shared
 * memory in a fixed order (bitwise reproducible). */
int ms_gemm_plan_fused_head(void* plan, const void* const* feat, const int32_t* inv, int inv_ld, int n_mod,
                            int feat_dim, int M, const void* W1, const float* b1, const void* W2, const float* b2,
                            int n_classes, float* logits, long long ldo);
/* The same head for small passes as ONE weight-streaming launch
 * (MODE_HEAD_GEMV): FC1 over 128 CTAs (4 hidden rows each, W1 chunks held in
 * registers, features gathered through inv, absent modality = zero K block)
 * -> bf16 h[M, 512] in `h` -> grid barrier on `sync` (two zeroed uint32
 * words, left zeroed/advanced for the next launch) -> FC2, one warp per
 * class.  Replaces the same reference fusion step as ms_gemm_plan_fused_head
 * (profile.py:157-159 drop rule, profile.py:170-174 head); K <= 4096. */
int ms_gemm_plan_head_gemv(void* plan, const void* const* feat, const int32_t* inv, int inv_ld, int n_mod,
                           int feat_dim, int M, const void* W1, const float* b1, const void* W2, const float* b2,
                           int n_classes, float* logits, long long ldo, void* h, void* sync);
/* Fuse a 1x1 conv (64 -> 64, + bias + ReLU; BN-Inception's conv2_red) into a
 * stem plan (output width <= 112): the pooled rows become the A operand of a
 * second tcgen05 MMA in the same kernel and Y receives the 1x1's output
 * (rows of ldy at y_col0); the pooled map itself is not stored.  Wred: the
 * [64 out, 64 in] bf16 weights pre-swizzled to the SW128 K-major layout
 * (encoders.pack_sw128_weight). */
int ms_gemm_plan_stem_set_reduce(void* plan, const void* Wred, const float* bias, void* Y, long long ldy, int y_col0);
int ms_gemm_plan_gather(void* plan, const void* const* feat, const int32_t* inv, int inv_ld, int n_mod,
                        int feat_dim, int M, const void* W, int N, int BN, const float* bias, int relu,
                        int out_fp32, void* D, long long ldd, int col0);
/* add a bf16 residual (same row mapping as the output, row stride res_ld)
 * after the activation: D = act(A W^T + b) + R */
int ms_gemm_plan_set_residual(void* plan, const void* residual, long long res_ld);
/* split K over `ksplit` CTAs per output tile (small-M GEMMs): each K part
 * stores its partial sums into its own slab of the caller's fp32 workspace
 * ws[ksplit, M, ws_ld] (ws_ld >= N, % 4 == 0); a finalize kernel adds the
 * slabs in part order (bitwise reproducible) and applies bias/activation/
 * residual; ms_gemm_run issues GEMM + finalize.  Dense/gather/conv
 * single-segment plans. */
int ms_gemm_plan_set_splitk(void* plan, int ksplit, float* ws, long long ws_ld);
int ms_gemm_run(const void* plan, void* stream);
/* run the plan as 2-CTA clusters on SM pairs (tcgen05.mma.cta_group::2,
 * 256-row tiles, half the weight rows per CTA); dense/conv bf16 plans
 * without split-K or residual */
int ms_gemm_plan_set_pair(void* plan, int enable);
/* profiling aid: bit0 = skip the epilogue stores (mainloop-only timing) */
int ms_gemm_plan_debug(void* plan, int flags);
/* Debug: per-CTA %globaltimer stamps (8 x u64 per CTA: entry, prologue done,
 * PDL wait done, first TMA issued, first data ready, last MMA commit, first
 * accumulator ready, epilogue done) into buf[grid_x * 8], or NULL to stop. */
int ms_gemm_plan_set_trace(void* plan, unsigned long long* buf);
int ms_gemm_plan_info(const void* plan, int* grid_x, int* grid_y, int* stages, int* smem_bytes);

/* ---- HBM-bound ops (NHWC bf16) ---------------------------------------- */
/* max (is_max=1) or average (count includes padding) pooling, k x k */
int ms_pool2d(const void* X, int n_img, int H, int W, int C, long long x_cstride, int k, int stride,
              int pad, int ceil_mode, int is_max, void* Y, long long y_cstride, int y_col0, void* stream);
/* as ms_pool2d, then y = act(pool + bias[c]) (bias fp32 or NULL, relu 0/1):
 * used for avgpool(proj(x)) + bias == proj(avgpool(x)) + bias, exact for
 * count-include-pad averaging, so the projection runs at the narrow width */
int ms_pool2d_ex(const void* X, int n_img, int H, int W, int C, long long x_cstride, int k, int stride,
                 int pad, int ceil_mode, int is_max, void* Y, long long y_cstride, int y_col0,
                 const float* bias, int relu, void* stream);
/* conv im2col for small-channel first layers: out[pixel, (kh*KW+kw)*C + c],
 * zero for columns >= KH*KW*C up to K_pad */
int ms_im2col(const void* X, int n_img, int H, int W, int C, int KH, int KW, int stride, int pad,
              void* out, int K_pad, void* stream);
/* global average pool + TSN segment consensus: X[(r*S + s)*HW + p, C] ->
 * Y[r, C] = mean over s, p */
int ms_segment_mean(const void* X, int n_req, int S, int HW, int C, void* Y, long long y_ld, void* stream);

/* ---- transformer towers (configs[2]: ViT-B/16 image + BERT-base text) --
 * ms_layernorm: Y[r] = LN(X[r]) * gamma + beta over C (C % 256 == 0), fp32
 *   statistics, arbitrary row strides (e.g. only the CLS rows).
 * ms_attention: per sequence s and head h, O = softmax(Q K^T * scale) V with
 *   qkv rows [Q | K | V] (H*64 each), row stride ld; O rows H*64, stride ldo.
 * ms_patchify: NHWC [n, S, S, C] -> [n*(S/P)^2, P*P*C] rows, K order (kh,kw,c).
 * ms_vit_embed: tok[s*L] = cls + pos[0]; tok[s*L+1+p] = pe[s*(L-1)+p] + pos[1+p].
 * ms_bert_embed: Y[t] = LN(word[ids[t]] + pos[t % L] + type0). */
int ms_layernorm(const void* X, long long ldx, long long rows, const float* gamma, const float* beta, void* Y,
                 long long ldy, int C, float eps, void* stream);
int ms_attention(const void* qkv, long long ld, int L, int H, int n_seq, void* out, long long ldo, float scale,
                 void* stream);
int ms_patchify(const void* X, int n, int S, int C, int P, void* Y, void* stream);
int ms_vit_embed(const void* pe, const void* cls, const void* pos, int n, int L, int D, void* tok, void* stream);
int ms_bert_embed(const int32_t* ids, long long n_tok, int L, const void* word, const void* pos, const void* type0,
                  const float* gamma, const float* beta, void* Y, int D, float eps, void* stream);

/* ---- op programs: a whole encoder forward as one native call ---------- */
int ms_op_gemm(void* op, const void* plan);
int ms_op_pool2d(void* op, const void* X, int n_img, int H, int W, int C, long long x_cstride, int k,
                 int stride, int pad, int ceil_mode, int is_max, void* Y, long long y_cstride, int y_col0);
int ms_op_pool2d_ex(void* op, const void* X, int n_img, int H, int W, int C, long long x_cstride, int k,
                    int stride, int pad, int ceil_mode, int is_max, void* Y, long long y_cstride, int y_col0,
                    const float* bias, int relu);
int ms_op_im2col(void* op, const void* X, int n_img, int H, int W, int C, int KH, int KW, int stride,
                 int pad, void* out, int K_pad);
int ms_op_segment_mean(void* op, const void* X, int n_req, int S, int HW, int C, void* Y, long long y_ld);
int ms_op_layernorm(void* op, const void* X, long long ldx, long long rows, const float* gamma, const float* beta,
                    void* Y, long long ldy, int C, float eps);
int ms_op_attention(void* op, const void* qkv, long long ld, int L, int H, int n_seq, void* out, long long ldo,
                    float scale);
int ms_op_patchify(void* op, const void* X, int n, int S, int C, int P, void* Y);
int ms_op_vit_embed(void* op, const void* pe, const void* cls, const void* pos, int n, int L, int D, void* tok);
int ms_op_bert_embed(void* op, const int32_t* ids, long long n_tok, int L, const void* word, const void* pos,
                     const void* type0, const float* gamma, const float* beta, void* Y, int D, float eps);
int ms_program_run(const void* ops, int n_ops, void* stream);

/* ---- profiler timing (CUDA events) ------------------------------------ */
int ms_event_create(void** ev);
int ms_event_destroy(void* ev);
int ms_event_record(void* ev, void* stream);
int ms_event_elapsed_us(void* start, void* stop, double* us);
/* 0 = completed, 1 = not yet, -1 = error (see ms_last_error) */
int ms_event_query(void* ev);
/* serving-loop plumbing without framework overhead: make `stream` wait for
 * `ev` (an ms_event), and launch an instantiated CUDA graph (the executor's
 * captured encoder / head graphs) on `stream` */
int ms_stream_wait_event(void* stream, void* ev);
int ms_graph_launch(void* graph_exec, void* stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* MOSEL_B200_H */
