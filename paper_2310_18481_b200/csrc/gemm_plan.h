// Plan and parameter structures shared by the GEMM translation units
// (gemm.cu: the generic tcgen05 GEMM / implicit-GEMM conv kernels and the
// fused stem; convpool.cu: the fused 3x3 conv + 3x3/2 max pool).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "mosel_b200.h"

namespace mosel {

constexpr int kEpiWarps = 8;                  // 2 per TMEM lane quarter
constexpr int kThreads = 64 + 32 * kEpiWarps;  // TMA + MMA + epilogue warps
constexpr int kMaxBias = 4096;  // staged bias floats (N <= 4096)
constexpr int kStageRowBytes = 80;                         // 64 B of bf16 + 16 B pad (conflict-free)
constexpr int kStageWarpBytes = 32 * kStageRowBytes;       // one warp's 32 x 32 bf16 chunk
constexpr int kStageBytes = kEpiWarps * kStageWarpBytes;   // epilogue staging buffers
constexpr int kBM = 128;
constexpr int kMaxHaloStages = 16;
constexpr int kBK = 64;
constexpr int kABytes = kBM * kBK * 2;  // 16 KB per stage

enum GemmMode : int {
  MODE_DENSE = 0, MODE_CONV = 1, MODE_GATHER = 2, MODE_CONV_SMALLC = 3, MODE_CONV_C4 = 5,
  MODE_CONV_HALO = 6, MODE_CONV_C12 = 7, MODE_CONV_K32 = 8, MODE_STEM_POOL = 9, MODE_CONV_POOL = 10,
  MODE_FUSED_HEAD = 11, MODE_HEAD_GEMV = 12
};
// MODE_CONV_K32: implicit-GEMM conv whose input channel count is a multiple
// of 32 but not of 64 (96, 160, 224): K runs over (tap, 32-channel part)
// halves, two per K block (SW64 boxes, like C4/C12), so K = 9 * Cin exactly
// instead of 9 * ceil64(Cin) (25 % / 17 % / 12.5 % fewer MMAs).
// MODE_CONV_C12: the 10-channel flow stack stored as 12-channel pixels (row
// and column padded like C4).  One filter row's window is 8 pixels x 12 ch =
// 96 elements = three 32-element SW64 boxes; K blocks take the 21 halves
// (row, part) two at a time (K 672 + 32 zero-weight, vs 896 for 16-channel
// pixels), consecutive output columns 48 B apart.
// MODE_CONV_HALO: 3x3 / stride 1 / pad 1 convolutions over images at least
// 14 pixels wide.  The output tile is bh whole image rows of P pixels (P =
// the image width + 2 rounded up to 8, so bh * P = 128).  Per 64-channel
// chunk ONE TMA box loads the (bh + 2) x P halo of input pixels (zero fill at
// the borders) into shared memory, and each of the 9 taps is an MMA whose A
// operand is the same tile read from a start address shifted by
// (dy * P + dx) rows of 128 B -- a K-major SW128 descriptor may start at any
// 128-B row (tools/umma_probe.py: the swizzle is address based), and 8-row
// groups stay 1024 B apart across halo rows because P is a multiple of 8.
// A traffic drops ~6x versus one box per tap; only the weights stream per
// tap.  Output columns >= OW (and rows >= OH) read wrapped halo pixels and
// are clipped by the TMA store.
// MODE_CONV_C4: stride-2 first convolutions over 4-channel pixels (rgb 3 ->
// 4, audio 1 -> 4) stored with `pad` zero rows AND columns around every
// frame.  One output pixel's KW-tap window in one input row is 8 pixels x 4
// channels = 64 contiguous bytes and consecutive output columns start 16
// bytes apart: a 4-D tensor map {window 32 elems (64 B), output column
// (16 B), padded input row (stride 2), image} with SWIZZLE_64B puts one
// filter row's windows for the whole tile in the UMMA K-major SW64 layout.  A
// K block = TWO filter rows = two such boxes in the two 8 KB halves of the
// stage (K 0-31 | 32-63): K = ceil(KH/2) blocks of 64 (7x7: 4 instead of the
// 7 of the 8-channel window mode -- 1.75x fewer MMAs, half the A bytes, and
// the gather writes 8-byte pixels instead of 16).
// MODE_CONV_SMALLC: first-layer convolutions with few channels (C8 = 8 or
// 16 stored channels).  The input is stored W-padded by `pad` zero pixels on
// each side, so for output pixel (oh, ow) and filter row kh the KW-tap
// window is one contiguous run of 8 pixels (8*C8 elements).  A 4-D tensor
// map whose innermost dimension IS that window and whose next dimension
// steps one output column (s pixels — the windows overlap) turns each
// 128-byte slice of a window into one smem row, so a K block = (kh, window
// half) is ONE TMA box in the standard SW128 K-major layout.  K order: (kh, j, c) with j < 8 (taps j >= KW are
// zero-weight).  Replaces an im2col round trip through HBM.

struct Seg {
  int n_begin, n_end;
  void* ptr;
  long long ldd;
  int col0;
  int flags;  // MS_SEG_NO_RELU
};

struct GemmParams {
  int mode;
  int M;       // DENSE/GATHER rows
  int m_tiles; // 128-row tiles (CONV: pixel blocks)
  int N;       // valid output columns
  int BN;      // tile width (multiple of 32, <= 256)
  int num_kb;  // K blocks
  int stages;
  int a_bytes;  // bytes of one A TMA box (CONV: bn*bh*bw*128)
  int b_bytes;
  // CONV geometry
  int n_img, OH, OW, stride, pad, KW, cchunks, bn, bh, bw, tiles_w, tiles_h;
  int smallc_halves, smallc_jpb;  // K blocks per filter row, window pixels per K block
  int pair;                       // 1: CTA-pair (cta_group::2) kernel
  // GATHER
  const __nv_bfloat16* feat[4];
  const int32_t* inv;  // [n_mod, inv_ld]
  int inv_ld, feat_dim, n_mod;
  // epilogue: v = act(acc + bias[n]) (+ residual[row, n])
  const float* bias;
  int relu, out_fp32, nseg, debug_flags;  // relu: activation MS_ACT_*; debug_flags bit0: skip stores
  const __nv_bfloat16* residual;   // same row mapping as the output, row stride res_ld
  long long res_ld;
  Seg seg[4];
  // split-K: tile = (m, n, k-part); partial sums -> fp32 workspace (atomics),
  // bias/act/convert applied by splitk_finalize_kernel
  int ksplit, kb_per;
  float* ws;
  long long ws_ld;
  unsigned long long* trace;  // debug: per-CTA %globaltimer stamps (kTraceSlots each) or null
  int tma_store;    // 1: bf16 epilogue writes each 128 x 32 chunk with one TMA store (StoreMaps)
  int halo_slot;    // MODE_CONV_HALO: bytes of one halo buffer (2 buffers precede the weight ring)
  int b_resident;   // MODE_CONV_HALO: all 9 x cchunks weight tiles stay in smem for the CTA's lifetime
  int warp_store;   // EPI_TMA: each epilogue warp stores its own 32 rows (no cross-warp barrier)
  int tile_groups;  // EPI_TMA, BN <= 64: the two epilogue warp groups take alternate tiles
  int direct_store; // EPI_TMA conv tiles: registers -> global, no smem staging (A/B only, MS_DIRECT_STORE:
                    // measured 13 % slower on conv2 at 56^2 than the TMA-store epilogue)
  int stage_bytes;  // epilogue staging bytes in shared memory
  int occ2;         // launch the 2-CTAs-per-SM instantiation (OCC = 2)
  int single_acc;   // one TMEM accumulator (occ2 plans with BN > 128)
  // MODE_STEM_POOL: raw pre-padded 4-channel input rows, fused 3x3/2 max pool
  const uint8_t* xraw;
  const uint8_t* wraw;  // MODE_STEM_POOL: row-pair weights (encoders.pack_stem_weight)
  long long x_plane;    // MODE_STEM_POOL with planes: bytes between 4-channel input planes
  int planes, plane_bytes;
  const uint8_t* red_w;   // MODE_STEM_POOL: fused 1x1 (64 -> 64) on the pooled rows, SW128 pre-swizzled weights
  const float* red_bias;  //   its bias; output = seg[1] (the pooled map itself is then not stored)
  long long x_pitch;   // bytes of one padded input row
  int Hp, PH, PW, units;
  __nv_bfloat16* hbuf;  // MODE_HEAD_GEMV: bf16 hidden rows [M, 512] (caller buffer)
};

// One bf16 output tensor map per epilogue segment (TMA stores, SWIZZLE_64B):
// DENSE/GATHER 2-D {cols, M} box {32, 128}; CONV 4-D {cols, OW, OH, n} box
// {32, bw, bh, bn}, so a conv tile's rows land at their (n, oh, ow) pixels and
// out-of-range rows/columns are clipped by the TMA unit.
struct alignas(64) StoreMaps {
  CUtensorMap m[4];
};
constexpr int kStoreChunkBytes = kBM * 64;            // 128 rows x 32 bf16
constexpr int kStoreBytes = 2 * kStoreChunkBytes;     // one chunk buffer per column group
constexpr int kTraceSlots = 12;

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define GEMM_TRACE(slot)                                                      \
  do {                                                                        \
    if (p.trace != nullptr) p.trace[blockIdx.x * kTraceSlots + (slot)] = gtimer(); \
  } while (0)

struct alignas(64) GemmPlan {
  CUtensorMap tmA;
  CUtensorMap tmB;
  StoreMaps tmD;
  GemmParams p;
  int grid_x, grid_y, smem_bytes, tmem_cols;
  const void* w_ptr;  // weight tensor (re-encoded for CTA-pair half boxes)
  long long w_kpad, w_rows;
};


int sm_count();
int launch_conv_pool(const GemmPlan* P, cudaStream_t stream);
int launch_fused_head(const GemmPlan* P, cudaStream_t stream);
int launch_head_gemv(const GemmPlan* P, cudaStream_t stream);

}  // namespace mosel
