// tcgen05/TMEM GEMM for the per-modality encoders and the fusion head.
//
//   D[m, n] = act( sum_k A[m, k] * W[n, k] + bias[n] )      bf16 in, fp32 acc
//
// One 128 x BN output tile per CTA (UMMA M=128, cta_group::1, N = BN <= 256),
// K in blocks of 64 bf16 (one 128-byte swizzle row).  Warp roles:
//   warp 0      : TMA producer (A and W tiles; W always by TMA)
//   warp 1      : TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2..5  : epilogue (TMEM -> regs -> bias/ReLU -> global); in
//                 GATHER mode they are also the A producers (cp.async)
// A-operand modes:
//   DENSE  : A is a row-major [M, K] matrix, 2-D TMA box {64, 128}
//   CONV   : implicit-GEMM convolution over NHWC input. The M tile is a
//            (bn images x bh rows x bw cols) block of output pixels; each
//            K block is one (tap, 64-channel chunk) and is ONE 4-D TMA box
//            {64, bw*s, bh*s, bn} with element strides {1, s, s, 1} at the
//            tap-shifted coordinate.  TMA zero-fills out-of-bounds
//            coordinates, which implements the convolution padding and the
//            channel tail for free.
//   GATHER : masked late-fusion concat.  Row i, K block kb reads modality
//            k = kb*64 / F from its compacted feature buffer at row inv_k[i];
//            absent modalities (inv = -1) are zero-filled — exactly
//            "skipping those K columns".
// The epilogue routes 32-column chunks to up to 4 destination segments so
// merged 1x1 branch GEMMs write straight into Inception concat slices.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "mosel_b200.h"
#include "gemm_plan.h"
#include "ptx.cuh"
#include "runtime.h"

namespace mosel {

// exact-form GELU, 0.5 x (1 + erf(x / sqrt 2)), with erf from Abramowitz &
// Stegun 7.1.26 (|error| <= 1.5e-7, below bf16 output rounding by ~4 orders):
// one MUFU reciprocal + one MUFU exp2 + 9 FMA-class ops and no branches,
// where libdevice erff took ~25 instructions with divergent ranges and made
// the ViT/BERT FC1 epilogue-bound (tools/vqa_gemm.py: 729 vs 1151 TF/s
// without the activation at M=18912 N=3072 K=768)
__device__ __forceinline__ float gelu_erf(float x) {
  const float z = fabsf(x) * 0.70710678118654752f;
  float t, e;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(fmaf(0.3275911f, z, 1.0f)));
  float q = fmaf(t, 1.061405429f, -1.453152027f);
  q = fmaf(t, q, 1.421413741f);
  q = fmaf(t, q, -0.284496736f);
  q = fmaf(t, q, 0.254829592f);
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-z * z * 1.4426950408889634f));
  const float erf_abs = fmaf(-q * t, e, 1.0f);
  const float erf_x = copysignf(erf_abs, x);
  return 0.5f * x * (1.0f + erf_x);
}

__device__ __forceinline__ float activate(float x, int act) {
  switch (act) {
    case MS_ACT_RELU: return fmaxf(x, 0.0f);
    case MS_ACT_GELU: return gelu_erf(x);
    case MS_ACT_TANH: return tanhf(x);
    default: return x;
  }
}

template <int ACT>
__device__ __forceinline__ void convert_chunk(const uint32_t (&v)[32], const float* bch, uint32_t (&pk)[16]) {
#pragma unroll
  for (int j = 0; j < 16; ++j)
    pk[j] = pack_bf16x2(activate(__uint_as_float(v[2 * j]) + bch[2 * j], ACT),
                        activate(__uint_as_float(v[2 * j + 1]) + bch[2 * j + 1], ACT));
}

struct TileIdx {
  int m, n, kb0, kb1;
};
// PAIR: t enumerates (m pair, n) tiles; CTA `rank` of the pair owns M tile
// 2 * pair + rank (the peer of an odd last pair reads and writes nothing:
// its boxes lie wholly out of bounds -- TMA zero-fills / clips them)
template <int PAIR>
__device__ __forceinline__ TileIdx decode_tile(const GemmParams& p, int t, int n_tiles, uint32_t rank) {
  TileIdx r;
  if (PAIR) {
    const int mp = t / n_tiles;
    r.m = 2 * mp + (int)rank;
    r.n = t - mp * n_tiles;
    r.kb0 = 0;
    r.kb1 = p.num_kb;
    return r;
  }
  const int kp = t % p.ksplit;
  const int mn = t / p.ksplit;
  r.m = mn / n_tiles;
  r.n = mn - r.m * n_tiles;
  r.kb0 = kp * p.kb_per;
  r.kb1 = min(p.num_kb, r.kb0 + p.kb_per);
  return r;
}

// Epilogue flavours (template parameter EPI):
//   EPI_TMA    bf16 output, each 128 x 32 chunk staged (SW64) and written by one
//              TMA store per 32-column chunk; up to 4 segments; optional residual
//   EPI_F32    fp32 output, direct per-thread stores (logits heads)
//   EPI_SPLITK fp32 partial sums -> workspace atomics (finalize applies bias/act)
enum GemmEpi : int { EPI_TMA = 0, EPI_F32 = 1, EPI_SPLITK = 2 };

template <int ACT>
__device__ __forceinline__ void convert_chunk4(const uint32_t (&v)[32], const float* bch, uint32_t (&pk)[16]) {
  const float4* b4 = reinterpret_cast<const float4*>(bch);
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const float4 b = b4[q];
    pk[2 * q] = pack_bf16x2(activate(__uint_as_float(v[4 * q]) + b.x, ACT),
                            activate(__uint_as_float(v[4 * q + 1]) + b.y, ACT));
    pk[2 * q + 1] = pack_bf16x2(activate(__uint_as_float(v[4 * q + 2]) + b.z, ACT),
                                activate(__uint_as_float(v[4 * q + 3]) + b.w, ACT));
  }
}

// One kernel instantiation per (A-operand mode, epilogue, activation): each
// carries only its own code (the generic kernel's every-mode/every-activation
// epilogue was instruction-latency bound at ~1 us per 32-column chunk).
//
// PAIR = 1: CTA-pair variant (clusters of 2 on an SM pair,
// tcgen05.mma.cta_group::2, M = 256 per instruction).  Each CTA loads its own
// 128-row A block (or halo) and HALF of the BN weight rows, so the weight
// bytes each SM pulls from L2 halve (the 3x3 convs below 56^2 are L2-read
// bound: ~42 B/clk/SM with every SM loading, MEASURED_PEAKS / B300 notes), and
// an N <= 96 MMA is no longer A-operand SMEM-read bound.  Protocol:
//   full[s], afull[h] (leader) : one arrive.expect_tx of BOTH CTAs' bytes; the
//                                peer's TMA completes on the leader's barrier
//   empty[s], aempty[h], tfull : multicast tcgen05.commit from the leader
//   tempty[a] (leader)         : both CTAs' epilogue warps arrive (remote)
// OCC = 2: an instantiation capped at 96 registers, so that two CTAs (of this
// or another op of a concurrent Inception branch lane) fit on one SM when the
// plan also keeps its shared memory <= ~113 KB and its TMEM <= 256 columns
// (GemmParams::occ2; tools/ab.sh MS_OCC2=1).
template <int MODE, int EPI, int ACT, int PAIR, int OCC = 1>
__global__ void __launch_bounds__(kThreads, OCC)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ GemmParams p, const __grid_constant__ StoreMaps tmD) {
  // Persistent: CTA b processes tiles b, b + grid, ...; tile t -> (m = t / n_tiles,
  // n = t % n_tiles).  The smem ring (full/empty) and the two TMEM accumulator
  // buffers (tfull/tempty) carry their phases across tiles, so the TMA
  // producer prefetches the next tile while the epilogue drains this one.
  constexpr bool kConv = MODE == MODE_CONV || MODE == MODE_CONV_SMALLC || MODE == MODE_CONV_C4 ||
                          MODE == MODE_CONV_HALO || MODE == MODE_CONV_C12 || MODE == MODE_CONV_K32;
  if (threadIdx.x == 0) GEMM_TRACE(0);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // align inside the shared window without leaving the shared address space
  // (a uintptr_t round trip would turn every smem access into a generic LD)
  uint8_t* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
  const int stages = p.stages;
  uint8_t* smA = smem;
  uint8_t* smB = smem + (MODE == MODE_CONV_HALO ? 2 * p.halo_slot : stages * kABytes);
  uint8_t* sstage = smB + stages * p.b_bytes;  // [p.stage_bytes], 1024-B aligned
  uint64_t* full = reinterpret_cast<uint64_t*>(sstage + p.stage_bytes);
  uint64_t* empty = full + stages;
  uint64_t* tfull = empty + stages;
  uint64_t* tempty = tfull + 2;
  uint64_t* afull = tempty + 2;   // MODE_CONV_HALO halo buffers
  uint64_t* aempty = afull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aempty + 2);
  float* sbias = reinterpret_cast<float*>(tmem_slot + 4);  // [N], 16-B aligned

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n_tiles = (p.N + p.BN - 1) / p.BN;
  const uint32_t rank = PAIR ? cluster_ctarank() : 0u;
  const bool leader = rank == 0;
  const int num_tiles = PAIR ? ((p.m_tiles + 1) / 2) * n_tiles : p.m_tiles * n_tiles * p.ksplit;
  const int cta0 = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;  // this CTA's (pair's) first tile
  const int ncta = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  // the leader's barrier for a pair's shared completions (own barrier otherwise)

  if (threadIdx.x == 0) {
    const uint32_t full_count = (MODE == MODE_GATHER) ? 1 + 128 : 1;
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], full_count);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      // one arrive per epilogue warp (per warp of the owning group with tile
      // groups), from both CTAs of a pair
      mbar_init(&tempty[a], ((EPI == EPI_TMA && MODE != MODE_GATHER && p.tile_groups) ? kEpiWarps / 2 : kEpiWarps) *
                                (PAIR ? 2 : 1));
      mbar_init(&afull[a], 1);
      mbar_init(&aempty[a], 1);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    if (MODE != MODE_GATHER) tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  uint32_t acc_stride = 32;
  while (acc_stride < (uint32_t)p.BN) acc_stride <<= 1;
  // two accumulators (the epilogue of tile i overlaps the MMAs of tile i+1), one
  // for a wide-N plan launched two CTAs per SM (the co-resident CTA fills the gap)
  const int n_acc = p.single_acc ? 1 : 2;
  const uint32_t tmem_cols = (uint32_t)n_acc * acc_stride;
  if (warp == 1) {
    if (PAIR)
      tmem_alloc_pair(tmem_slot, tmem_cols);
    else
      tmem_alloc(tmem_slot, tmem_cols);
  }
  const int nb_pad = (p.N + 31) & ~31;
  for (int i = threadIdx.x; i < nb_pad && i < kMaxBias; i += blockDim.x)
    sbias[i] = (p.bias != nullptr && i < p.N) ? p.bias[i] : 0.0f;
  tc_fence_before();
  if (PAIR)
    cluster_sync_all();  // barrier inits + TMEM allocation visible to the pair
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // PDL: this prologue overlapped the previous kernel's tail.  Trigger only
  // once TMEM is held: a dependent CTA that allocated first on this SM while
  // waiting for us would otherwise deadlock our tcgen05.alloc.
  if (threadIdx.x == 0) GEMM_TRACE(1);
  pdl_trigger();
  pdl_wait();
  if (threadIdx.x == 0) GEMM_TRACE(2);

  if (warp == 0) {
    if (MODE == MODE_CONV_HALO && lane == 0) {
      // ------------------------------------- TMA producer (halo + per-tap weights)
      int s = 0, hs = 0;
      uint32_t phase = 0, hphase = 0;
      if (p.b_resident) {  // this CTA's N tile of weights once, before the first halo
        // (grid is a multiple of n_tiles, so every tile t of this CTA has n = t % n_tiles fixed)
        const int n_tile = cta0 % n_tiles;
        if (leader) mbar_arrive_expect_tx(&full[0], 9 * p.cchunks * p.b_bytes * (PAIR ? 2 : 1));
        for (int kb = 0; kb < 9 * p.cchunks; ++kb) {
          if (PAIR)
            tma_load_2d_pair(smem_addr(smB + kb * p.b_bytes), &tmB, &full[0], kb * kBK,
                             n_tile * p.BN + (int)rank * (p.BN / 2));
          else
            tma_load_2d(smem_addr(smB + kb * p.b_bytes), &tmB, &full[0], kb * kBK, n_tile * p.BN);
        }
      }
      for (int t = cta0; t < num_tiles; t += ncta) {
        const TileIdx ti = decode_tile<PAIR>(p, t, n_tiles, rank);
        const int th = ti.m % p.tiles_h;
        const int img = ti.m / p.tiles_h;
        for (int cc = 0; cc < p.cchunks; ++cc) {
          mbar_wait(&aempty[hs], hphase ^ 1);
          if (t == cta0 && cc == 0) GEMM_TRACE(3);
          if (PAIR) {
            if (leader) mbar_arrive_expect_tx(&afull[hs], 2 * p.a_bytes);
            tma_load_4d_pair(smem_addr(smA + hs * p.halo_slot), &tmA, &afull[hs], cc * kBK, -1, th * p.bh - 1, img);
          } else {
            mbar_arrive_expect_tx(&afull[hs], p.a_bytes);
            tma_load_4d(smem_addr(smA + hs * p.halo_slot), &tmA, &afull[hs], cc * kBK, -1, th * p.bh - 1, img);
          }
          if (p.b_resident) {
            if (++hs == 2) {
              hs = 0;
              hphase ^= 1;
            }
            continue;
          }
          for (int tap = 0; tap < 9; ++tap) {
            mbar_wait(&empty[s], phase ^ 1);
            if (PAIR) {
              if (leader) mbar_arrive_expect_tx(&full[s], 2 * p.b_bytes);
              tma_load_2d_pair(smem_addr(smB + s * p.b_bytes), &tmB, &full[s], (tap * p.cchunks + cc) * kBK,
                               ti.n * p.BN + (int)rank * (p.BN / 2));
            } else {
              mbar_arrive_expect_tx(&full[s], p.b_bytes);
              tma_load_2d(smem_addr(smB + s * p.b_bytes), &tmB, &full[s], (tap * p.cchunks + cc) * kBK,
                          ti.n * p.BN);
            }
            if (++s == stages) {
              s = 0;
              phase ^= 1;
            }
          }
          if (++hs == 2) {
            hs = 0;
            hphase ^= 1;
          }
        }
      }
    } else if (MODE != MODE_CONV_HALO && lane == 0) {
      // ------------------------------------------------ TMA producer
      int s = 0;
      uint32_t phase = 0;
      const uint32_t tx = (MODE == MODE_GATHER ? 0 : p.a_bytes) + p.b_bytes;
      for (int t = cta0; t < num_tiles; t += ncta) {
        const TileIdx ti = decode_tile<PAIR>(p, t, n_tiles, rank);
        const int m_tile = ti.m, n_tile = ti.n;
        int n0 = 0, oh0 = 0, ow0 = 0;
        if constexpr (kConv) {
          const int tw = m_tile % p.tiles_w;
          const int th = (m_tile / p.tiles_w) % p.tiles_h;
          const int tn = m_tile / (p.tiles_w * p.tiles_h);
          n0 = tn * p.bn;
          oh0 = th * p.bh * p.stride - p.pad;
          ow0 = tw * p.bw * p.stride - p.pad;
        }
        for (int kb = ti.kb0; kb < ti.kb1; ++kb) {
          mbar_wait(&empty[s], phase ^ 1);
          const uint32_t a_dst = smem_addr(smA + s * kABytes);
          const uint32_t b_dst = smem_addr(smB + s * p.b_bytes);
          if (PAIR) {
            if (leader) mbar_arrive_expect_tx(&full[s], 2 * tx);
          } else {
            mbar_arrive_expect_tx(&full[s], tx);
          }
          if constexpr (MODE == MODE_DENSE) {
            if (PAIR)
              tma_load_2d_pair(a_dst, &tmA, &full[s], kb * kBK, m_tile * kBM);
            else
              tma_load_2d(a_dst, &tmA, &full[s], kb * kBK, m_tile * kBM);
          } else if constexpr (MODE == MODE_CONV) {
            const int tap = kb / p.cchunks;
            const int cc = kb - tap * p.cchunks;
            const int kh = tap / p.KW;
            const int kw = tap - kh * p.KW;
            if (PAIR)
              tma_load_4d_pair(a_dst, &tmA, &full[s], cc * kBK, ow0 + kw, oh0 + kh, n0);
            else
              tma_load_4d(a_dst, &tmA, &full[s], cc * kBK, ow0 + kw, oh0 + kh, n0);
          } else if constexpr (MODE == MODE_CONV_SMALLC) {
            const int kh = kb / p.smallc_halves;
            const int half = kb - kh * p.smallc_halves;
            // ow0/oh0 already include -pad; W is pre-padded in memory so the
            // column coordinate is the raw output column
            tma_load_4d(a_dst, &tmA, &full[s], half * kBK, (ow0 + p.pad) / p.stride, oh0 + kh, n0);
          } else if constexpr (MODE == MODE_CONV_C4) {
            // padded input row of (output row oh, filter row 2kb + l) = 2*oh + 2kb + l
            const int c2 = (ow0 + p.pad) / 2, r0 = oh0 + p.pad + 2 * kb;
            tma_load_4d(a_dst, &tmA, &full[s], 0, c2, r0, n0);
            tma_load_4d(a_dst + kABytes / 2, &tmA, &full[s], 0, c2, r0 + 1, n0);
          } else if constexpr (MODE == MODE_CONV_C12) {
            // halves h = 2kb, 2kb+1 of the (filter row, 32-element part) sequence;
            // the one past the last (zero weights) re-reads a valid box
            const int c2 = (ow0 + p.pad) / 2;
#pragma unroll
            for (int l = 0; l < 2; ++l) {
              const int h = min(2 * kb + l, p.smallc_halves - 1);
              const int row = h / 3, part = h - 3 * (h / 3);
              tma_load_4d(a_dst + l * (kABytes / 2), &tmA, &full[s], part * 32, c2, oh0 + p.pad + row, n0);
            }
          } else if constexpr (MODE == MODE_CONV_K32) {
            // halves (tap, 32-channel part), two per K block; past the end: a valid box (zero weights)
            const int parts = p.cchunks;  // 32-channel parts per tap
#pragma unroll
            for (int l = 0; l < 2; ++l) {
              const int h = min(2 * kb + l, 9 * parts - 1);
              const int tap = h / parts, part = h - tap * parts;
              const int kh = tap / 3, kw = tap - 3 * (tap / 3);
              if (PAIR)
                tma_load_4d_pair(a_dst + l * (kABytes / 2), &tmA, &full[s], part * 32, ow0 + kw, oh0 + kh, n0);
              else
                tma_load_4d(a_dst + l * (kABytes / 2), &tmA, &full[s], part * 32, ow0 + kw, oh0 + kh, n0);
            }
          }
          if (PAIR)
            tma_load_2d_pair(b_dst, &tmB, &full[s], kb * kBK, n_tile * p.BN + (int)rank * (p.BN / 2));
          else
            tma_load_2d(b_dst, &tmB, &full[s], kb * kBK, n_tile * p.BN);
          if (t == cta0 && kb == ti.kb0) GEMM_TRACE(3);
          if (++s == stages) {
            s = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1 && MODE == MODE_CONV_HALO && leader) {
    // ------------------------------------ MMA issuer: 9 shifted views per halo
    const uint32_t idesc = PAIR ? umma_idesc_bf16_m256((uint32_t)p.BN) : umma_idesc_bf16_m128((uint32_t)p.BN);
    int s = 0, hs = 0;
    uint32_t phase = 0, hphase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    const int P = p.bw;
    if (p.b_resident) {
      mbar_wait(&full[0], 0);
      tc_fence_after();
    }
    for (int t = cta0; t < num_tiles; t += ncta) {
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + (uint32_t)acc * acc_stride;
      for (int cc = 0; cc < p.cchunks; ++cc) {
        mbar_wait(&afull[hs], hphase);
        tc_fence_after();
        if (lane == 0 && t == cta0 && cc == 0) GEMM_TRACE(4);
        if (lane == 0 && t + ncta >= num_tiles && cc == p.cchunks - 1) GEMM_TRACE(5);
        const uint32_t halo = smem_addr(smA + hs * p.halo_slot);
        if (p.b_resident) {  // 9 taps straight from the resident weights
          if (lane == 0) {
#pragma unroll 1
            for (int tap = 0; tap < 9; ++tap) {
              const int dy = tap / 3, dx = tap - 3 * (tap / 3);
              const uint64_t adesc = umma_desc_sw128(halo + (uint32_t)((dy * P + dx) * 128));
              const uint64_t bdesc = umma_desc_sw128(smem_addr(smB + (tap * p.cchunks + cc) * p.b_bytes));
#pragma unroll
              for (int k = 0; k < kBK / 16; ++k) {
                if (PAIR)
                  umma_bf16_pair(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (cc | tap | k) != 0);
                else
                  umma_bf16(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (cc | tap | k) != 0);
              }
            }
            if (PAIR) {
              umma_commit_pair(&aempty[hs], 0x3);
              if (cc == p.cchunks - 1) umma_commit_pair(&tfull[acc], 0x3);
            } else {
              umma_commit(&aempty[hs]);
              if (cc == p.cchunks - 1) umma_commit(&tfull[acc]);
            }
          }
          __syncwarp();
          if (++hs == 2) {
            hs = 0;
            hphase ^= 1;
          }
          continue;
        }
        for (int tap = 0; tap < 9; ++tap) {
          mbar_wait(&full[s], phase);
          tc_fence_after();
          if (lane == 0) {
            const int dy = tap / 3, dx = tap - 3 * (tap / 3);
            const uint64_t adesc = umma_desc_sw128(halo + (uint32_t)((dy * P + dx) * 128));
            const uint64_t bdesc = umma_desc_sw128(smem_addr(smB + s * p.b_bytes));
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {
              if (PAIR)
                umma_bf16_pair(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (cc | tap | k) != 0);
              else
                umma_bf16(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (cc | tap | k) != 0);
            }
            if (PAIR) {
              umma_commit_pair(&empty[s], 0x3);
              if (tap == 8) {
                umma_commit_pair(&aempty[hs], 0x3);
                if (cc == p.cchunks - 1) umma_commit_pair(&tfull[acc], 0x3);
              }
            } else {
              umma_commit(&empty[s]);
              if (tap == 8) {
                umma_commit(&aempty[hs]);
                if (cc == p.cchunks - 1) umma_commit(&tfull[acc]);
              }
            }
          }
          __syncwarp();
          if (++s == stages) {
            s = 0;
            phase ^= 1;
          }
        }
        if (++hs == 2) {
          hs = 0;
          hphase ^= 1;
        }
      }
      if (++acc == n_acc) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  } else if (warp == 1 && MODE != MODE_CONV_HALO && leader) {
    // -------------------------------------------------- MMA issuer
    const uint32_t idesc = PAIR ? umma_idesc_bf16_m256((uint32_t)p.BN) : umma_idesc_bf16_m128((uint32_t)p.BN);
    int s = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = cta0; t < num_tiles; t += ncta) {
      const TileIdx ti = decode_tile<PAIR>(p, t, n_tiles, rank);
      mbar_wait(&tempty[acc], acc_phase ^ 1);  // epilogue drained this buffer
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + (uint32_t)acc * acc_stride;
      for (int kb = ti.kb0; kb < ti.kb1; ++kb) {
        mbar_wait(&full[s], phase);
        tc_fence_after();
        if constexpr (MODE == MODE_GATHER) fence_proxy_async_smem();
        if (lane == 0 && t == cta0 && kb == ti.kb0) GEMM_TRACE(4);
        if (lane == 0) {
          const uint64_t bdesc = umma_desc_sw128(smem_addr(smB + s * p.b_bytes));
          if constexpr (MODE == MODE_CONV_C4 || MODE == MODE_CONV_C12 || MODE == MODE_CONV_K32) {  // 2 SW64 halves
            const uint32_t a0 = smem_addr(smA + s * kABytes);
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {
              const uint64_t adesc = umma_desc_sw64(a0 + (k >> 1) * (kABytes / 2)) + 2 * (k & 1);
              if (PAIR)
                umma_bf16_pair(d_tmem, adesc, bdesc + 2 * k, idesc, (kb != ti.kb0) || k != 0);
              else
                umma_bf16(d_tmem, adesc, bdesc + 2 * k, idesc, (kb != ti.kb0) || k != 0);
            }
          } else {
            const uint64_t adesc = umma_desc_sw128(smem_addr(smA + s * kABytes));
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {
              // +32 bytes per 16-element K step inside the swizzled row (>>4 = 2)
              if (PAIR)
                umma_bf16_pair(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb != ti.kb0) || k != 0);
              else
                umma_bf16(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb != ti.kb0) || k != 0);
            }
          }
          if (PAIR) {
            umma_commit_pair(&empty[s], 0x3);
            if (kb == ti.kb1 - 1) umma_commit_pair(&tfull[acc], 0x3);
          } else {
            umma_commit(&empty[s]);
            if (kb == ti.kb1 - 1) {
              umma_commit(&tfull[acc]);
              GEMM_TRACE(5);
            }
          }
        }
        __syncwarp();
        if (++s == stages) {
          s = 0;
          phase ^= 1;
        }
      }
      if (++acc == n_acc) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  } else if (warp >= 2) {
    // ---------------------- warps 2..9: gather (2..5) + epilogue (all 8)
    const int q = warp & 3;               // TMEM lane quarter of this warp
    const int grp = (warp - 2) >> 2;      // column-chunk group: chunks c with c % 2 == grp
    const int r = q * 32 + lane;          // tile row owned by this thread
    const bool issuer = (warp == 2 + 4 * grp) && lane == 0;  // EPI_TMA store issuer
    uint8_t* sbuf = sstage + grp * kStoreChunkBytes;         // EPI_TMA chunk buffer
    uint8_t* srow = sbuf + r * 64;
    const int sw = (r >> 1) & 3;  // SWIZZLE_64B phase of this row
    int s = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    // tile groups (narrow tiles, BN <= 64): the two warp groups take
    // alternate tiles (group g = accumulator g) and all of a tile's chunks,
    // so two tiles' epilogues run at once instead of one tile's two halves
    const bool tg = EPI == EPI_TMA && MODE != MODE_GATHER && p.tile_groups;
    const int cs = tg ? 1 : 2;  // chunk step
    // a pair's accumulator-empty barriers live in the leader CTA
    const uint32_t tempty_bar0 = PAIR ? mapa_shared(smem_addr(&tempty[0]), 0) : 0u;
    for (int t = cta0; t < num_tiles; t += ncta) {
      if (tg && acc != grp) {  // the other group's tile
        if (++acc == n_acc) {
          acc = 0;
          acc_phase ^= 1;
        }
        continue;
      }
      const TileIdx ti = decode_tile<PAIR>(p, t, n_tiles, rank);
      const int m_tile = ti.m, n_tile = ti.n;
      if constexpr (MODE == MODE_GATHER) {
        if (grp == 0) {
          const int row = m_tile * kBM + r;
          const int kb_per_mod = p.feat_dim / kBK;
          for (int kb = ti.kb0; kb < ti.kb1; ++kb) {
            mbar_wait(&empty[s], phase ^ 1);
            const int k = kb / kb_per_mod;
            const int off = (kb - k * kb_per_mod) * kBK;
            const __nv_bfloat16* src = nullptr;
            if (row < p.M) {
              const int j = p.inv[(long long)k * p.inv_ld + row];
              if (j >= 0) src = p.feat[k] + (long long)j * p.feat_dim + off;
            }
            const uint32_t dst = smem_addr(smA + s * kABytes) + r * 128;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const uint32_t phys = (uint32_t)(c ^ (r & 7));
              cp_async_16(dst + phys * 16, src ? (const void*)(src + c * 8) : (const void*)p.feat[0],
                          src ? 16u : 0u);
            }
            cp_async_mbar_arrive_noinc(&full[s]);
            if (++s == stages) {
              s = 0;
              phase ^= 1;
            }
          }
        }
      }

      // output row for this thread (or -1): residual / fp32 / split-K paths
      long long out_row = -1;
      if constexpr (kConv) {
        if (EPI != EPI_TMA || p.residual != nullptr || p.direct_store) {
          const int tw = m_tile % p.tiles_w;
          const int th = (m_tile / p.tiles_w) % p.tiles_h;
          const int tn = m_tile / (p.tiles_w * p.tiles_h);
          const int per_img = p.bh * p.bw;
          if (r < p.bn * per_img) {
            const int i = r / per_img;
            const int y = (r - i * per_img) / p.bw;
            const int x = r - i * per_img - y * p.bw;
            const int n = tn * p.bn + i, oh = th * p.bh + y, ow = tw * p.bw + x;
            if (n < p.n_img && oh < p.OH && ow < p.OW) out_row = ((long long)n * p.OH + oh) * p.OW + ow;
          }
        }
      } else {
        const int row = m_tile * kBM + r;
        if (row < p.M) out_row = row;
      }

      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      if (warp == 2 && lane == 0 && t == cta0) GEMM_TRACE(6);
      const uint32_t t_base = tmem_base + (uint32_t)acc * acc_stride + ((uint32_t)(q * 32) << 16);
      const int n_first = n_tile * p.BN;
      const int n_chunks = (min(p.BN, p.N - n_first) + 31) >> 5;
      // chunks c = grp, grp + 2, ...: TMEM loads double-buffered so chunk c+2's
      // load is in flight while chunk c is converted and stored
      auto release_acc = [&]() {  // every TMEM read of this accumulator has completed
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (PAIR)
            mbar_arrive_cluster(tempty_bar0 + (uint32_t)acc * 8u);
          else
            mbar_arrive(&tempty[acc]);
        }
      };
      auto process = [&](const uint32_t (&v)[32], int c) {
        const int nb = n_first + c * 32;
        const bool tr0 = warp == 2 && lane == 0 && t == cta0 && c == grp;
        if (tr0) GEMM_TRACE(8);
        if constexpr (EPI == EPI_SPLITK) {
          // this K part's partial sums -> its own workspace slab (plain stores;
          // the finalize adds the slabs in part order: deterministic)
          if (out_row >= 0) {
            float* w = p.ws + ((long long)(ti.kb0 / p.kb_per) * p.M + out_row) * p.ws_ld + nb;
#pragma unroll
            for (int j = 0; j < 32; j += 4)
              if (nb + j < p.N)
                *reinterpret_cast<float4*>(w + j) =
                    make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]), __uint_as_float(v[j + 2]),
                                __uint_as_float(v[j + 3]));
          }
        } else if constexpr (EPI == EPI_F32) {
          if (out_row >= 0) {
            const Seg& S = p.seg[0];
            float* dst = reinterpret_cast<float*>(S.ptr) + out_row * S.ldd + S.col0 - S.n_begin + nb;
            const float* bch = sbias + nb;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (nb + j < p.N) dst[j] = activate(__uint_as_float(v[j]) + bch[j], ACT);
          }
        } else {  // EPI_TMA
          if (p.debug_flags & 1) return;  // debug: accumulate only (no convert / store)
          int g = 0;
#pragma unroll
          for (int gg = 1; gg < 4; ++gg)
            if (gg < p.nseg && nb >= p.seg[gg].n_begin) g = gg;
          uint32_t pk[16];
          if (p.seg[g].flags & MS_SEG_NO_RELU)
            convert_chunk4<MS_ACT_NONE>(v, sbias + nb, pk);
          else
            convert_chunk4<ACT>(v, sbias + nb, pk);
          if (p.residual != nullptr && out_row >= 0) {
            const __nv_bfloat16* rp = p.residual + out_row * p.res_ld + nb;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              if (nb + 2 * j < p.N) {  // pairs never straddle N (N is even)
                const __nv_bfloat162 a2 = *reinterpret_cast<const __nv_bfloat162*>(&pk[j]);
                const __nv_bfloat162 r2 = *reinterpret_cast<const __nv_bfloat162*>(rp + 2 * j);
                pk[j] = pack_bf16x2(__bfloat162float(a2.x) + __bfloat162float(r2.x),
                                    __bfloat162float(a2.y) + __bfloat162float(r2.y));
              }
            }
          }
          if (tr0) GEMM_TRACE(9);
          if (p.direct_store) {
            // registers -> global (64 contiguous bytes per row): no shared-memory
            // staging traffic competing with the MMAs' operand reads
            if (out_row >= 0) {
              const Seg& S = p.seg[g];
              __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(S.ptr) + out_row * S.ldd + S.col0 + (nb - S.n_begin);
#pragma unroll
              for (int j = 0; j < 4; ++j)
                if (nb + 8 * j < S.n_end)
                  *reinterpret_cast<uint4*>(dst + 8 * j) = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
            }
            return;
          }
          if (p.warp_store) {
            // this warp's 32 rows x 32 columns: own 2 KB slice, own TMA store,
            // no barrier with the other warps of the group
            if (lane == 0) bulk_wait_read0();  // my previous store has read my slice
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 4; ++j)
              *reinterpret_cast<uint4*>(srow + ((j ^ sw) << 4)) =
                  make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              const int c0 = nb - p.seg[g].n_begin;
              const uint32_t src = smem_addr(sbuf + q * 32 * 64);
              if constexpr (kConv) {
                const int tw = m_tile % p.tiles_w;
                const int th = (m_tile / p.tiles_w) % p.tiles_h;
                const int tn = m_tile / (p.tiles_w * p.tiles_h);
                const int r0 = q * 32;
                if (r0 < p.bh * p.bw) {
                  const int x = tw * p.bw + (p.bw >= 32 ? r0 % p.bw : 0);
                  const int y = th * p.bh + r0 / p.bw;
                  tma_store_4d(&tmD.m[g], src, c0, x, y, tn * p.bn);
                }
              } else {
                tma_store_2d(&tmD.m[g], src, c0, m_tile * kBM + q * 32);
              }
              bulk_commit();
            }
            return;
          }
          if (issuer) bulk_wait_read0();  // the previous chunk's store has read the buffer
          named_bar_sync(1 + grp, 128);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            *reinterpret_cast<uint4*>(srow + ((j ^ sw) << 4)) =
                make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
          fence_proxy_async_smem();
          named_bar_sync(1 + grp, 128);
          if (issuer) {
            const int c0 = nb - p.seg[g].n_begin;
            if constexpr (kConv) {
              const int tw = m_tile % p.tiles_w;
              const int th = (m_tile / p.tiles_w) % p.tiles_h;
              const int tn = m_tile / (p.tiles_w * p.tiles_h);
              tma_store_4d(&tmD.m[g], smem_addr(sbuf), c0, tw * p.bw, th * p.bh, tn * p.bn);
            } else {
              tma_store_2d(&tmD.m[g], smem_addr(sbuf), c0, m_tile * kBM);
            }
            bulk_commit();
            if (tr0) GEMM_TRACE(10);
          }
        }
      };
      int c = tg ? 0 : grp;
      if constexpr (OCC == 2) {
        // 96-register instantiation: one TMEM buffer (the double-buffered
        // loads below spilled 280 B per thread here; the OCC=2 epilogue waits
        // on its accumulator anyway, so the load latency is not exposed)
        uint32_t va[32];
        for (; c < n_chunks; c += cs) {
          tmem_ld_32x32b_x32(t_base + (uint32_t)(c * 32), va);
          tmem_wait_ld();
          if (c + cs >= n_chunks) release_acc();
          process(va, c);
        }
      } else {
      uint32_t va[32], vb[32];
      if (c < n_chunks) tmem_ld_32x32b_x32(t_base + (uint32_t)(c * 32), va);
      while (c < n_chunks) {
        tmem_wait_ld();
        if (c + cs < n_chunks)
          tmem_ld_32x32b_x32(t_base + (uint32_t)((c + cs) * 32), vb);
        else
          release_acc();
        process(va, c);
        c += cs;
        if (c >= n_chunks) break;
        tmem_wait_ld();
        if (c + cs < n_chunks)
          tmem_ld_32x32b_x32(t_base + (uint32_t)((c + cs) * 32), va);
        else
          release_acc();
        process(vb, c);
        c += cs;
      }
      }
      if (!tg && grp >= n_chunks) release_acc();  // no chunk for this group in a narrow tile
      if (warp == 2 && lane == 0 && t == cta0) GEMM_TRACE(11);
      if (++acc == n_acc) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (EPI == EPI_TMA && (issuer || (p.warp_store && lane == 0))) bulk_wait0();
    if (warp == 2 && lane == 0) GEMM_TRACE(7);
  }
  if (PAIR) {
    tc_fence_before();
    cluster_sync_all();  // the leader's MMAs into the peer's TMEM are complete
    if (warp == 1) {
      tc_fence_after();
      tmem_dealloc_pair(tmem_base, tmem_cols);
    }
  } else {
    __syncthreads();
    if (warp == 1) {
      tc_fence_after();
      tmem_dealloc(tmem_base, tmem_cols);
    }
  }
}

typedef void (*GemmKernelFn)(const CUtensorMap, const CUtensorMap, const GemmParams, const StoreMaps);

template <int MODE, int EPI, int PAIR = 0>
static GemmKernelFn pick_act(int act) {
  switch (act) {
    case MS_ACT_RELU: return gemm_tc_kernel<MODE, EPI, MS_ACT_RELU, PAIR>;
    case MS_ACT_GELU: return gemm_tc_kernel<MODE, EPI, MS_ACT_GELU, PAIR>;
    case MS_ACT_TANH: return gemm_tc_kernel<MODE, EPI, MS_ACT_TANH, PAIR>;
    default: return gemm_tc_kernel<MODE, EPI, MS_ACT_NONE, PAIR>;
  }
}

// The instantiation for a plan (null if the combination is unsupported).
static GemmKernelFn gemm_kernel_for(const GemmParams& p) {
  if (p.occ2 && !p.pair && p.ksplit <= 1 && !p.out_fp32 && p.tma_store && p.relu == MS_ACT_RELU) {
    switch (p.mode) {
      case MODE_DENSE: return gemm_tc_kernel<MODE_DENSE, EPI_TMA, MS_ACT_RELU, 0, 2>;
      case MODE_CONV: return gemm_tc_kernel<MODE_CONV, EPI_TMA, MS_ACT_RELU, 0, 2>;
      case MODE_CONV_K32: return gemm_tc_kernel<MODE_CONV_K32, EPI_TMA, MS_ACT_RELU, 0, 2>;
      default: break;
    }
  }
  if (p.pair) {  // CTA pairs: bf16 TMA-store epilogue only (set_pair checks)
    switch (p.mode) {
      case MODE_DENSE: return pick_act<MODE_DENSE, EPI_TMA, 1>(p.relu);
      case MODE_CONV: return pick_act<MODE_CONV, EPI_TMA, 1>(p.relu);
      case MODE_CONV_K32: return pick_act<MODE_CONV_K32, EPI_TMA, 1>(p.relu);
      case MODE_CONV_HALO: return pick_act<MODE_CONV_HALO, EPI_TMA, 1>(p.relu);
      default: return nullptr;
    }
  }
  if (p.ksplit > 1) {
    if (p.mode == MODE_DENSE) return gemm_tc_kernel<MODE_DENSE, EPI_SPLITK, MS_ACT_NONE, 0>;
    if (p.mode == MODE_GATHER) return gemm_tc_kernel<MODE_GATHER, EPI_SPLITK, MS_ACT_NONE, 0>;
    if (p.mode == MODE_CONV) return gemm_tc_kernel<MODE_CONV, EPI_SPLITK, MS_ACT_NONE, 0>;
    return nullptr;
  }
  if (p.out_fp32) {
    if (p.mode == MODE_DENSE) return pick_act<MODE_DENSE, EPI_F32>(p.relu);
    if (p.mode == MODE_GATHER) return pick_act<MODE_GATHER, EPI_F32>(p.relu);
    return nullptr;
  }
  if (!p.tma_store) return nullptr;
  switch (p.mode) {
    case MODE_DENSE: return pick_act<MODE_DENSE, EPI_TMA>(p.relu);
    case MODE_CONV: return pick_act<MODE_CONV, EPI_TMA>(p.relu);
    case MODE_GATHER: return pick_act<MODE_GATHER, EPI_TMA>(p.relu);
    case MODE_CONV_SMALLC: return pick_act<MODE_CONV_SMALLC, EPI_TMA>(p.relu);
    case MODE_CONV_C4: return pick_act<MODE_CONV_C4, EPI_TMA>(p.relu);
    case MODE_CONV_HALO: return pick_act<MODE_CONV_HALO, EPI_TMA>(p.relu);
    case MODE_CONV_C12: return pick_act<MODE_CONV_C12, EPI_TMA>(p.relu);
    case MODE_CONV_K32: return pick_act<MODE_CONV_K32, EPI_TMA>(p.relu);
    default: return nullptr;
  }
}


// ------------------------------------------------------------------------
// MODE_STEM_POOL: the 7x7/2 first convolution over 4-channel pixels (rgb 3 ->
// 4, audio 1 -> 4) FUSED with the 3x3/2 ceil-mode max pool that follows it.
// The unpooled conv output (4x the pooled bytes) never reaches HBM.
//
// A operand straight from the raw input rows: output pixel ow's window in a
// padded input row starts at byte 16*ow (stride 2 x 4 ch x 2 B) and is 32
// contiguous bf16 (8 pixels x 4 ch).  That is exactly the K-major
// SWIZZLE_NONE UMMA layout with 8-row x 16-B core matrices, LBO (K step
// between core matrices) = 16 B and SBO (8-row group step) = 128 B: core
// matrices overlap in memory, which the tensor core does not mind.  A conv
// row is 14 MMAs (M = 128 >= OW output pixels, N = 64, K = 16) on shifted
// descriptors into the rows brought in by ONE bulk copy -- no im2col, no
// overlapping TMA boxes.  Weights (64 x 256, K = (kh, 8 px, 4 ch), the C4
// packing) stay resident.
//
// Work: a CTA owns a contiguous range of pooled rows (image, i).  Pooled row i
// takes conv rows 2i..2i+2 and consecutive pooled rows share conv row 2i+2,
// so the CTA's walk is one tile per pooled row: CLOSE(i) = conv rows 2i+1 and
// 2i+2 (two accumulators of one 128-column TMEM slot, input rows 4i+2..4i+10
// in one bulk copy), preceded by OPEN(i) = conv row 2i where a run starts
// (the range's first row or an image's first row).  One producer / MMA /
// epilogue handshake per tile, not per conv row: the per-handshake barrier
// latency of the three single-threaded roles, not the MMAs, bounded the
// one-row-per-handshake version (measured: 122 us skeleton-bound).  The
// epilogue converts (bias, bf16), max-pools horizontally and keeps the
// vertical max in registers; ReLU is applied once to the pooled value (it
// commutes with max, as does the bf16 rounding: result == pool(bf16(relu(conv)))).
//
// kOverlap (output width <= 112): the A descriptor's 8-row-group stride is 7
// pixels (SBO 112 B) instead of 8, so consecutive row groups share one pixel
// and each warp's 32 TMEM lanes hold 29 consecutive conv pixels 28q..28q+28 --
// exactly the support of its 14 pooled pixels 14q..14q+13.  The horizontal
// pool is then two warp shuffles per register: no shared-memory row, no
// barrier between epilogue warps.  (M = 128 rows still buy 113 distinct
// pixels, as many as 112 linear rows.)  Otherwise (audio, 128 wide) the
// converted rows go through a swizzled shared-memory row buffer.
constexpr int kStemSlots = 4;              // TMEM slots of 128 columns (two conv rows)
constexpr int kStemKH = 7;                 // 7x7 filters (plan-checked)
constexpr int kStemMaxRows = 9;            // input rows of a CLOSE tile
constexpr int kStemWRow = 128 * 32 * 2;      // one input row's [W_j ; W_(j-2)]: 128 n x 32 k
constexpr int kStemWBytes = kStemMaxRows * kStemWRow;
constexpr int kStemWBlk = 64 * 32 * 2;      // planes variant: one (filter row, plane) 64 n x 32 k block
constexpr int kStemRowBuf = 128 * 128;     // <= 128 conv pixels x 64 ch bf16
#ifndef STEM_EPI_WARPS
#define STEM_EPI_WARPS 8
#endif
constexpr int kStemEpiWarps = STEM_EPI_WARPS;  // 2 per TMEM lane quarter, 32 channels each (8: 1.1x over 16 for rgb -- fewer warps competing with the MMA warp for issue slots)
constexpr int kStemCh = 64 / (kStemEpiWarps / 4);
// + one warp issuing the fused 1x1 conv (conv2_red) on the pooled rows (p.red_w)
constexpr int kStemThreads = 64 + 32 * kStemEpiWarps + 32;
constexpr int kStemRedWarp = 2 + kStemEpiWarps;
constexpr int kStemRedA = 128 * 128;     // one pooled row as the 1x1's A operand (SW128, 128 rows)
constexpr int kStemRedW = 64 * 128;      // the 1x1's 64 x 64 weights (SW128, pre-swizzled)
template <int N>
__device__ __forceinline__ void stem_tmem_ld(uint32_t taddr, uint32_t (&r)[N]) {
  if constexpr (N == 16)
    tmem_ld_32x32b_x16(taddr, r);
  else
    tmem_ld_32x32b_x32(taddr, r);
}

__device__ __forceinline__ uint32_t bf16x2_max(uint32_t a, uint32_t b) {
  __nv_bfloat162 r = __hmax2(*reinterpret_cast<__nv_bfloat162*>(&a), *reinterpret_cast<__nv_bfloat162*>(&b));
  return *reinterpret_cast<uint32_t*>(&r);
}
__device__ __forceinline__ uint4 bf16x8_max(uint4 a, uint4 b) {
  return make_uint4(bf16x2_max(a.x, b.x), bf16x2_max(a.y, b.y), bf16x2_max(a.z, b.z), bf16x2_max(a.w, b.w));
}

// The CTA's tile walk: units u0..u1-1, an OPEN tile before a unit that starts a
// run.  Tile = (img, i, open); conv rows: OPEN -> {2i}; CLOSE -> {2i+1, 2i+2 < OH}.
struct StemWalk {
  int u, u1, PH, OH, img, i;
  bool open;
  __device__ __forceinline__ void begin(int u0_, int u1_, int PH_, int OH_) {
    u1 = u1_; PH = PH_; OH = OH_; u = u0_;
    img = u / PH;  // the only division: later units step (img, i) incrementally
    i = u - img * PH;
    open = true;   // a run starts: conv row 2i is not carried over
  }
  __device__ __forceinline__ bool valid() const { return u < u1; }
  __device__ __forceinline__ void next() {
    if (open) { open = false; return; }  // OPEN(i) -> CLOSE(i)
    ++u;
    if (++i == PH) {
      i = 0;
      ++img;
      open = true;  // a new image starts a run
    }
  }
  __device__ __forceinline__ int row0() const { return open ? 2 * i : 2 * i + 1; }
  __device__ __forceinline__ int nrows() const { return open ? 1 : (2 * i + 2 < OH ? 2 : 1); }
};

template <bool kOverlap, int kPlanes>
__global__ void __launch_bounds__(kStemThreads, 1)
    stem_pool_kernel(const __grid_constant__ GemmParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
  const int stages = p.stages;
  const int a_stride = p.b_bytes;  // bytes per stage (9 padded input rows, 128-B rounded)
  uint8_t* smW = smem;
  constexpr int kWBytes = kPlanes == 1 ? kStemWBytes : kStemKH * kPlanes * kStemWBlk;
  uint8_t* smA = smW + kWBytes;
  uint8_t* rbuf = smA + stages * a_stride + 256;  // + slack: rows >= OW of the last tap read past a stage
  // fused 1x1 (red): two pooled-row A tiles + its weights, 1024-B aligned
  uint8_t* redA = smem + (((rbuf + (kOverlap ? 0 : kStemRowBuf)) - smem + 1023) & ~1023);
  uint8_t* redW = redA + 2 * kStemRedA;
  const bool red = kOverlap && p.red_w != nullptr;
  uint64_t* full = reinterpret_cast<uint64_t*>(red ? redW + kStemRedW : rbuf + (kOverlap ? 0 : kStemRowBuf));
  uint64_t* empty = full + stages;
  uint64_t* wbar = empty + stages;
  uint64_t* tfull = wbar + 1;
  uint64_t* tempty = tfull + kStemSlots;
  uint64_t* a_full = tempty + kStemSlots;  // red: pooled row b written (epilogue warps)
  uint64_t* r_full = a_full + 2;           // red: 1x1 of row b done (commit)
  uint64_t* r_empty = r_full + 2;          // red: TMEM result b drained (epilogue warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(r_empty + 2);
  float* sbias = reinterpret_cast<float*>(tmem_slot + 4);
  float* sbias_red = sbias + 64;
  // TMEM: conv slots of 128 columns (4, or 3 with the fused 1x1) + 2 x 64 for the 1x1
  const int slots = red ? 3 : kStemSlots;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int OH = p.OH, OW = p.OW, PH = p.PH, PW = p.PW;
  const int u0 = (int)((long long)p.units * blockIdx.x / gridDim.x);
  const int u1 = (int)((long long)p.units * (blockIdx.x + 1) / gridDim.x);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(wbar, 1);
    for (int s = 0; s < kStemSlots; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], kStemEpiWarps);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&a_full[b], kStemEpiWarps);
      mbar_init(&r_full[b], 1);
      mbar_init(&r_empty[b], kStemEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  if (threadIdx.x < 64) sbias[threadIdx.x] = p.bias ? p.bias[threadIdx.x] : 0.0f;
  if (threadIdx.x < 64) sbias_red[threadIdx.x] = (red && p.red_bias) ? p.red_bias[threadIdx.x] : 0.0f;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_trigger();  // after the TMEM allocation (see gemm_tc_kernel)
  if (warp == 0 && lane == 0) {  // weights are constants: load them before waiting on the producer grid
    mbar_arrive_expect_tx(wbar, kWBytes + (red ? kStemRedW : 0));
    for (int o = 0; o < kWBytes; o += 8192)
      bulk_load(smem_addr(smW + o), p.wraw + o, min(8192, kWBytes - o), wbar);
    if (red) bulk_load(smem_addr(redW), p.red_w, kStemRedW, wbar);
  }
  pdl_wait();

  StemWalk w;
  w.begin(u0, u1, PH, OH);
  // debug: CTA 0's first 32 tiles, stamps (MMA ready, MMA issued, epilogue ready, epilogue done)
  auto trace = [&](int k, int slot_) {
    if (p.trace != nullptr && blockIdx.x == 0 && k < 32) p.trace[k * 8 + slot_] = gtimer();
  };
  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------- producer
      int s = 0, kp = 0;
      uint32_t phase = 0;
      for (; w.valid(); w.next(), ++kp) {
        // conv rows row0 .. row0+n-1 read padded input rows 2*row0 .. 2*(row0+n-1)+6
        const uint32_t bytes = (uint32_t)((2 * w.nrows() + 5) * p.x_pitch);
        mbar_wait(&empty[s], phase ^ 1);
        trace(kp, 4);
        mbar_arrive_expect_tx(&full[s], bytes * kPlanes);
        const uint8_t* src = p.xraw + ((long long)w.img * p.Hp + 2 * w.row0()) * p.x_pitch;
#pragma unroll
        for (int pl = 0; pl < kPlanes; ++pl)
          bulk_load(smem_addr(smA + s * a_stride + pl * p.plane_bytes), src + pl * p.x_plane, bytes, &full[s]);
        if (++s == stages) {
          s = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {  // ------------------------------------ MMA issuer
    const uint32_t idesc = umma_idesc_bf16_m128(kPlanes == 1 ? 128 : 64);
    // descriptors built once: per (input row j, K half h) only the start-address
    // field moves (+(j - j0)*pitch + 32h bytes for A, +j*8 KB + 256h for B)
    const uint64_t a_desc0 = umma_desc_interleave(smem_addr(smA), 16, kOverlap ? 112 : 128);
    const uint64_t b_desc0 = umma_desc_interleave(smem_addr(smW), 128, 512);
    const uint32_t pitch16 = (uint32_t)(p.x_pitch >> 4), stage16 = (uint32_t)(a_stride >> 4);
    mbar_wait(wbar, 0);
    tc_fence_after();
    int s = 0, k = 0;
    uint32_t phase = 0;
    for (; w.valid(); w.next(), ++k) {
      const int slot = k % slots;
      const int n = w.nrows();
      mbar_wait(&tempty[slot], (uint32_t)(((k / slots) & 1) ^ 1));
      mbar_wait(&full[s], phase);
      tc_fence_after();
      if (lane == 0) trace(k, 0);
      {
        // the conv-row pair (r, r+1): OPEN = (2i-1, 2i) needs input rows j = 2..8
        // only, CLOSE = (2i+1, 2i+2) rows 0..8 (0..6 when 2i+2 is past the map).
        // Warp-uniform issue (elect.sync inside each instruction): the issuing
        // warp shares its scheduler with busy epilogue warps, so every
        // instruction on this path costs.
        const uint64_t ad = a_desc0 + (uint64_t)(s * stage16);
        const uint32_t d = tmem_base + (uint32_t)(slot * 128);
        const int j0 = w.open ? 2 : 0, j1 = j0 + 2 * n + 4;
        const uint32_t a_lo = (uint32_t)ad, a_hi = (uint32_t)(ad >> 32);
        const uint32_t b_lo = (uint32_t)b_desc0, b_hi = (uint32_t)(b_desc0 >> 32);
        if constexpr (kPlanes == 1) {
          for (int j = j0; j <= j1; ++j)
            umma_bf16_x2_elect(d, a_lo + (uint32_t)(j - j0) * pitch16, a_hi, b_lo + (uint32_t)j * (kStemWRow / 16),
                               b_hi, 16, idesc, j != j0);
        } else {
          // channel planes: per conv row, N = 64 MMAs over (filter row, plane);
          // weights W[kh][plane] 64 x 32 blocks (encoders.pack_stem_weight_planes)
          const uint32_t plane16 = (uint32_t)(p.plane_bytes >> 4);
          for (int dr = 0; dr < n; ++dr) {
            const uint32_t dd = d + (uint32_t)(w.open ? 64 : 64 * dr);
            const uint32_t ar = a_lo + (uint32_t)(2 * dr) * pitch16;
            for (int kh = 0; kh < kStemKH; ++kh)
#pragma unroll
              for (int pl = 0; pl < kPlanes; ++pl)
                umma_bf16_x2_elect(dd, ar + (uint32_t)kh * pitch16 + (uint32_t)pl * plane16, a_hi,
                                   b_lo + (uint32_t)((kh * kPlanes + pl) * (kStemWBlk / 16)), b_hi, 16, idesc,
                                   (kh | pl) != 0);
          }
        }
        umma_commit_elect(&empty[s]);
        umma_commit_elect(&tfull[slot]);
        if (lane == 0) trace(k, 1);
      }
      if (++s == stages) {
        s = 0;
        phase ^= 1;
      }
    }
  } else if (warp == kStemRedWarp) {  // ----------------- fused 1x1 (conv2_red) issuer
    if (red) {
      const uint32_t idesc = umma_idesc_bf16_m128(64);
      const uint64_t bdesc = umma_desc_sw128(smem_addr(redW));
      mbar_wait(wbar, 0);
      int kc = 0;  // CLOSE tiles
      for (; w.valid(); w.next()) {
        if (w.open) continue;
        const int b = kc & 1;
        mbar_wait(&a_full[b], (uint32_t)((kc >> 1) & 1));        // pooled row written
        mbar_wait(&r_empty[b], (uint32_t)(((kc >> 1) & 1) ^ 1));  // result b drained
        tc_fence_after();
        const uint64_t adesc = umma_desc_sw128(smem_addr(redA + b * kStemRedA));
        const uint32_t d = tmem_base + (uint32_t)(slots * 128 + 64 * b);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) umma_bf16_elect(d, adesc + 2 * kk, bdesc + 2 * kk, idesc, kk != 0);
        umma_commit_elect(&r_full[b]);
        ++kc;
      }
    }
  } else if constexpr (kOverlap) {  // ------------- epilogue warps (overlapping row groups)
    const int q = warp & 3, c = (warp - 2) >> 2;  // TMEM lane quarter, kStemCh-channel chunk
    const int x = 7 * (lane >> 3) + (lane & 7);   // this lane's conv pixel within the warp's 29
    auto lane_of = [](int y) { return y < 28 ? (y / 7) * 8 + y % 7 : 31; };
    const int src1 = lane_of(min(x + 1, 28)), src2 = lane_of(min(x + 2, 28));
    const int jj = x >> 1;                          // pooled pixel (local) when this lane owns one
    const bool owner = (lane & 7) < 7 && (x & 1) == 0 && x <= 26 && 14 * q + jj < PW;
    const bool three = 28 * q + x + 2 < OW;         // ceil mode: the last window may be 2 wide
    const Seg& Y = p.seg[0];
    const uint32_t t_lane = tmem_base + (uint32_t)(c * kStemCh) + ((uint32_t)(q * 32) << 16);
    const float* bch = sbias + c * kStemCh;
    uint32_t carry[kStemCh / 2];  // conv row 2i of the open pooled row, bf16(acc + bias), per pixel
    // fused 1x1: the pooled row of CLOSE tile kc goes to redA[kc & 1]; its 1x1
    // result is drained (bias, ReLU, bf16 -> p.red_y) while the next tile runs
    int kc = 0, prev_img = 0, prev_i = 0;
    const Seg& R = p.seg[1];
    auto drain = [&](int kd, int img_, int i_) {
      const int b = kd & 1;
      mbar_wait(&r_full[b], (uint32_t)((kd >> 1) & 1));
      tc_fence_after();
      uint32_t v[32];
      tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(slots * 128 + 64 * b + 32 * c), v);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&r_empty[b]);
      const int px = 32 * q + lane;  // pooled pixel = TMEM lane
      if (px < PW) {
        __nv_bfloat16* yr = reinterpret_cast<__nv_bfloat16*>(R.ptr) +
                            (((long long)img_ * PH + i_) * PW + px) * R.ldd + R.col0 + 32 * c;
        const float* br = sbias_red + 32 * c;
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          uint32_t o[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int e = 8 * g + 2 * t;
            o[t] = pack_bf16x2(fmaxf(__uint_as_float(v[e]) + br[e], 0.0f), fmaxf(__uint_as_float(v[e + 1]) + br[e + 1], 0.0f));
          }
          *reinterpret_cast<uint4*>(yr + 8 * g) = make_uint4(o[0], o[1], o[2], o[3]);
        }
      }
    };
    for (int k = 0; w.valid(); w.next(), ++k) {
      const int slot = k % slots;
      const int n = w.nrows();
      mbar_wait(&tfull[slot], (uint32_t)((k / slots) & 1));
      tc_fence_after();
      if (warp == 2 && lane == 0) trace(k, 2);
      uint32_t v0[kStemCh], v1[kStemCh];
      // OPEN: row 2i is the pair's second row (columns 64..127)
      stem_tmem_ld(t_lane + (uint32_t)(slot * 128 + (w.open ? 64 : 0)), v0);
      if (n == 2) stem_tmem_ld(t_lane + (uint32_t)(slot * 128 + 64), v1);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[slot]);
      if (w.open) {  // conv row 2i opens pooled row i
#pragma unroll
        for (int e = 0; e < kStemCh / 2; ++e)
          carry[e] = pack_bf16x2(__uint_as_float(v0[2 * e]) + bch[2 * e], __uint_as_float(v0[2 * e + 1]) + bch[2 * e + 1]);
        continue;
      }
      // CLOSE: vertical max of rows 2i, 2i+1 (, 2i+2) per pixel, then the
      // horizontal 3-max across lanes; row 2i+2 opens pooled row i+1
      __nv_bfloat16* y = reinterpret_cast<__nv_bfloat16*>(Y.ptr) +
                         (((long long)w.img * PH + w.i) * PW + 14 * q + jj) * Y.ldd + Y.col0 + c * kStemCh;
      const int pp = 14 * q + jj;  // pooled pixel = the 1x1's A row
      uint8_t* arow = redA + (kc & 1) * kStemRedA + pp * 128;
      if (red && kc >= 1) drain(kc - 1, prev_img, prev_i);  // frees redA[kc & 1] (the 1x1 of kc - 2 read it)
#pragma unroll
      for (int g = 0; g < kStemCh / 8; ++g) {
        uint32_t o[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int e = 4 * g + t;
          uint32_t m = bf16x2_max(carry[e], pack_bf16x2(__uint_as_float(v0[2 * e]) + bch[2 * e],
                                                        __uint_as_float(v0[2 * e + 1]) + bch[2 * e + 1]));
          if (n == 2) {
            const uint32_t r2 = pack_bf16x2(__uint_as_float(v1[2 * e]) + bch[2 * e],
                                            __uint_as_float(v1[2 * e + 1]) + bch[2 * e + 1]);
            m = bf16x2_max(m, r2);
            carry[e] = r2;
          }
          const uint32_t m1 = __shfl_sync(0xffffffffu, m, src1);
          const uint32_t m2 = __shfl_sync(0xffffffffu, m, src2);
          uint32_t h = bf16x2_max(m, m1);
          if (three) h = bf16x2_max(h, m2);
          o[t] = bf16x2_max(h, 0u);  // ReLU
        }
        if (owner) {
          if (red)
            *reinterpret_cast<uint4*>(arow + (((c * (kStemCh / 8) + g) ^ (pp & 7)) << 4)) = make_uint4(o[0], o[1], o[2], o[3]);
          else
            *reinterpret_cast<uint4*>(y + 8 * g) = make_uint4(o[0], o[1], o[2], o[3]);
        }
      }
      if (red) {  // this tile's pooled row -> the 1x1 issuer
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&a_full[kc & 1]);
        prev_img = w.img;
        prev_i = w.i;
        ++kc;
      }
      if (warp == 2 && lane == 0) trace(k, 3);
    }
    if (red && kc >= 1) drain(kc - 1, prev_img, prev_i);
  } else {  // ----------------------------- epilogue warps (linear rows, smem horizontal pool)
    const int q = warp & 3, c = (warp - 2) >> 2;  // TMEM lane quarter, kStemCh-channel chunk
    const int ow = q * 32 + lane;
    const int tid = threadIdx.x - 64;             // 0 .. 32 * kStemEpiWarps - 1
    const int n_items = PW * 8;                   // pooled pixels x 8 16-B channel groups
    const Seg& Y = p.seg[0];
    const uint32_t t_lane = tmem_base + (uint32_t)(c * kStemCh) + ((uint32_t)(q * 32) << 16);
    const float* bch = sbias + c * kStemCh;
    uint32_t carry[kStemCh / 2];
    for (int k = 0; w.valid(); w.next(), ++k) {
      const int slot = k % slots;
      const int n = w.nrows();
      mbar_wait(&tfull[slot], (uint32_t)((k / slots) & 1));
      tc_fence_after();
      uint32_t v0[kStemCh], v1[kStemCh];
      // OPEN: row 2i is the pair's second row (columns 64..127)
      stem_tmem_ld(t_lane + (uint32_t)(slot * 128 + (w.open ? 64 : 0)), v0);
      if (n == 2) stem_tmem_ld(t_lane + (uint32_t)(slot * 128 + 64), v1);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[slot]);
      if (w.open) {
#pragma unroll
        for (int e = 0; e < kStemCh / 2; ++e)
          carry[e] = pack_bf16x2(__uint_as_float(v0[2 * e]) + bch[2 * e], __uint_as_float(v0[2 * e + 1]) + bch[2 * e + 1]);
        continue;
      }
      // vertical max per pixel -> the row buffer (swizzled 16-B groups)
      uint32_t m[kStemCh / 2];
#pragma unroll
      for (int e = 0; e < kStemCh / 2; ++e) {
        m[e] = bf16x2_max(carry[e], pack_bf16x2(__uint_as_float(v0[2 * e]) + bch[2 * e],
                                                __uint_as_float(v0[2 * e + 1]) + bch[2 * e + 1]));
        if (n == 2) {
          const uint32_t r2 = pack_bf16x2(__uint_as_float(v1[2 * e]) + bch[2 * e],
                                          __uint_as_float(v1[2 * e + 1]) + bch[2 * e + 1]);
          m[e] = bf16x2_max(m[e], r2);
          carry[e] = r2;
        }
      }
      if (ow < OW) {
        uint8_t* row = rbuf + ow * 128;
#pragma unroll
        for (int t = 0; t < kStemCh / 8; ++t)
          *reinterpret_cast<uint4*>(row + ((((c * (kStemCh / 8) + t) ^ (ow & 7))) << 4)) =
              make_uint4(m[4 * t], m[4 * t + 1], m[4 * t + 2], m[4 * t + 3]);
      }
      named_bar_sync(1, 32 * kStemEpiWarps);
      __nv_bfloat16* yrow = reinterpret_cast<__nv_bfloat16*>(Y.ptr) + ((long long)w.img * PH + w.i) * PW * Y.ldd + Y.col0;
      for (int it = tid; it < n_items; it += 32 * kStemEpiWarps) {
        const int j = it >> 3, g = it & 7;
        const int x0 = 2 * j;
        const uint8_t* b0 = rbuf + x0 * 128;
        uint4 h = bf16x8_max(*reinterpret_cast<const uint4*>(b0 + ((g ^ (x0 & 7)) << 4)),
                             *reinterpret_cast<const uint4*>(b0 + 128 + ((g ^ ((x0 + 1) & 7)) << 4)));
        if (x0 + 2 < OW) h = bf16x8_max(h, *reinterpret_cast<const uint4*>(b0 + 256 + ((g ^ ((x0 + 2) & 7)) << 4)));
        *reinterpret_cast<uint4*>(yrow + (long long)j * Y.ldd + 8 * g) = bf16x8_max(h, make_uint4(0, 0, 0, 0));
      }
      named_bar_sync(1, 32 * kStemEpiWarps);  // rbuf is rewritten by the next CLOSE tile
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

// split-K finalize: D = act(sum_k ws[k] + bias) (+ residual), bf16 or fp32,
// one thread per 4 columns; the K-part slabs are added in part order, so the
// result is bitwise reproducible (no atomics, no workspace zeroing).
__global__ void splitk_finalize_kernel(const __grid_constant__ GemmParams p) {
  pdl_trigger();
  pdl_wait();
  const int n4 = (p.N + 3) / 4;
  const long long total = (long long)p.M * n4;
  const Seg& S = p.seg[0];
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long row = t / n4;
    const int n = (int)(t - row * n4) * 4;
    float av[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    for (int k = 0; k < p.ksplit; ++k) {
      const float4 a = *reinterpret_cast<const float4*>(p.ws + ((long long)k * p.M + row) * p.ws_ld + n);
      av[0] += a.x;
      av[1] += a.y;
      av[2] += a.z;
      av[3] += a.w;
    }
    for (int j = 0; j < 4 && n + j < p.N; ++j) {
      float x = activate(av[j] + (p.bias ? p.bias[n + j] : 0.0f), p.relu);
      if (p.residual) x += __bfloat162float(p.residual[row * p.res_ld + n + j]);
      const long long o = row * S.ldd + S.col0 + n + j - S.n_begin;
      if (p.out_fp32)
        reinterpret_cast<float*>(S.ptr)[o] = x;
      else
        reinterpret_cast<__nv_bfloat16*>(S.ptr)[o] = __float2bfloat16_rn(x);
    }
  }
}

// ==================================================================== host

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (fn == nullptr) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  return fn;
}

static int encode_map(CUtensorMap* m, int rank, const void* base, const cuuint64_t* dims,
                      const cuuint64_t* strides_bytes, const cuuint32_t* box, const cuuint32_t* estride,
                      CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  EncodeTiledFn fn = encode_fn();
  if (fn == nullptr) return set_error(MS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (no CUDA driver)");
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), dims, strides_bytes, box,
                  estride, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char msg[160];
    snprintf(msg, sizeof msg, "cuTensorMapEncodeTiled failed (%d) rank=%d", (int)r, rank);
    return set_error(MS_ERR_INVALID, msg);
  }
  return MS_OK;
}

int encode_bf16_map(CUtensorMap* m, int rank, const void* base, const cuuint64_t* dims,
                    const cuuint64_t* strides_bytes, const cuuint32_t* box, const cuuint32_t* estride,
                    CUtensorMapSwizzle swz) {
  return encode_map(m, rank, base, dims, strides_bytes, box, estride, swz);
}

int g_occ2_grid = -1;  // ms_set_occ2_grid (< 0: MS_OCC2_GRID / default)

int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
  }
  return n;
}

// pipeline depth cap (MS_MAX_STAGES: probe switch for tools/mainloop_probe.py)
static int max_stages() {
  const char* e = getenv("MS_MAX_STAGES");
  const int v = e ? atoi(e) : 0;
  return v >= 2 ? v : 8;
}

static int finish_plan(GemmPlan* P, const void* W, int K_pad, int N_rows_w, int BN, int num_kb, int grid_x) {
  GemmParams& p = P->p;
  if (BN % 32 != 0 || BN < 32 || BN > 256) return set_error(MS_ERR_INVALID, "BN must be a multiple of 32 in [32, 256]");
  if (p.N > kMaxBias) return set_error(MS_ERR_INVALID, "N exceeds the staged-bias capacity (4096)");
  if (K_pad % kBK != 0) return set_error(MS_ERR_INVALID, "weight K must be padded to a multiple of 64");
  cuuint64_t dims[2] = {(cuuint64_t)K_pad, (cuuint64_t)N_rows_w};
  cuuint64_t strides[1] = {(cuuint64_t)K_pad * 2};
  cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)BN};
  cuuint32_t es[2] = {1, 1};
  P->w_ptr = W;
  P->w_kpad = K_pad;
  P->w_rows = N_rows_w;
  int rc = encode_map(&P->tmB, 2, W, dims, strides, box, es);
  if (rc) return rc;
  p.BN = BN;
  static const bool no_tile_groups = getenv("MS_NO_TILE_GROUPS") != nullptr;  // A/B switch for tools
  static const int tg_max_bn = getenv("MS_TILE_GROUPS_BN") ? atoi(getenv("MS_TILE_GROUPS_BN")) : 64;
  p.tile_groups = (!no_tile_groups && BN <= tg_max_bn && p.mode != MODE_GATHER && !p.out_fp32) ? 1 : 0;
  p.num_kb = num_kb;
  p.ksplit = 1;
  p.kb_per = num_kb;
  p.b_bytes = BN * kBK * 2;
  const int per_stage = kABytes + p.b_bytes;
  const int bias_bytes = ((p.N + 31) / 32) * 32 * 4;
  p.stage_bytes = p.tma_store ? kStoreBytes : 0;  // fp32 / split-K epilogues stage nothing
  // 227 KB usable: 1 KB alignment slack, barriers, epilogue staging, bias
  int stages = (226 * 1024 - 1024 - 288 - p.stage_bytes - bias_bytes) / per_stage;
  if (stages > max_stages()) stages = max_stages();
  if (stages > num_kb) stages = num_kb < 2 ? 2 : num_kb;
  // two CTAs per SM (see gemm_tc_kernel's OCC): TMEM <= 256 columns, <= 112 KB of
  // shared memory (>= 2 stages: with a co-resident CTA, 2 stages per CTA beat
  // 3+ stages at one CTA per SM -- served-pass encoders -4.2 %,
  // profiles/r02_ab_two_ctas_per_sm.txt; MS_OCC2_MIN_STAGES for A/B)
  static const bool occ2_env = getenv("MS_OCC2") == nullptr || atoi(getenv("MS_OCC2")) != 0;  // default on
  const int per_occ2 = (112 * 1024 - 1024 - p.stage_bytes - (2 * 3 + 8) * 8 - 16 - bias_bytes) / per_stage;
  static const bool occ2_wide = getenv("MS_OCC2_NARROW") == nullptr;  // A/B: BN <= 128 plans only
  static const int occ2_min_stages = getenv("MS_OCC2_MIN_STAGES") ? atoi(getenv("MS_OCC2_MIN_STAGES")) : 2;
  // ... and only for layers with enough tiles to fill the GPU: a small pass's
  // kernels are latency-bound per CTA, where the full-stage, full-register
  // instantiation wins (MS_OCC2_MIN_TILES, default 64: best of 0/24/64/148 at
  // every pass size 1..96, profiles/r02_pass_sizes_occ2.txt)
  static const int occ2_min_tiles = getenv("MS_OCC2_MIN_TILES") ? atoi(getenv("MS_OCC2_MIN_TILES")) : 64;
  const int tiles_all = grid_x * ((p.N + BN - 1) / BN);
  p.occ2 = (occ2_env && tiles_all >= occ2_min_tiles && (BN <= 128 || occ2_wide) && per_occ2 >= occ2_min_stages &&
            p.tma_store && !p.out_fp32 &&
            p.relu == MS_ACT_RELU && (p.mode == MODE_DENSE || p.mode == MODE_CONV || p.mode == MODE_CONV_K32))
               ? 1
               : 0;
  p.single_acc = (p.occ2 && BN > 128) ? 1 : 0;  // TMEM: 2 x 128 or 1 x 256 columns per CTA
  if (p.occ2 && stages > per_occ2) stages = per_occ2;
  p.stages = stages;
  P->smem_bytes = 1024 + stages * per_stage + p.stage_bytes + (2 * stages + 8) * 8 + 16 + bias_bytes;
  if (P->smem_bytes > 227 * 1024) return set_error(MS_ERR_INVALID, "GEMM plan exceeds 227 KB shared memory");
  p.m_tiles = grid_x;
  const int tiles = grid_x * ((p.N + BN - 1) / BN);
  // up to two of this kernel's own CTAs per SM (MS_OCC2_GRID / ms_set_occ2_grid:
  // 0 never, 2 only with >= 4 tiles per SM, default 1 always: a kernel with no
  // concurrent partner still fills both slots -- single-encoder passes 3-6 %
  // faster, profiles/r02_abn_occ2.txt; with other encoders running beside it,
  // 2 leaves them the second slot -- mixed passes 0.7-3.4 % faster,
  // profiles/r02_ringab_grid2.txt; the executor plans both variants)
  const int occ2_grid = g_occ2_grid >= 0 ? g_occ2_grid : (getenv("MS_OCC2_GRID") ? atoi(getenv("MS_OCC2_GRID")) : 1);
  const bool grid2 = p.occ2 && (occ2_grid == 1 || (occ2_grid == 2 && tiles >= 4 * sm_count()));
  const int max_ctas = grid2 ? 2 * sm_count() : sm_count();
  P->grid_x = tiles < max_ctas ? tiles : max_ctas;
  P->grid_y = 1;
  int tc = 32;
  while (tc < BN) tc <<= 1;
  P->tmem_cols = (p.single_acc ? 1 : 2) * tc;
  return MS_OK;
}

static int encode_store_maps(GemmPlan* P) {
  GemmParams& p = P->p;
  p.tma_store = 0;
  if (p.out_fp32) return MS_OK;
  const bool conv = p.mode == MODE_CONV || p.mode == MODE_CONV_SMALLC || p.mode == MODE_CONV_C4 ||
                    p.mode == MODE_CONV_HALO || p.mode == MODE_CONV_C12 || p.mode == MODE_CONV_K32;
  // per-warp stores (each epilogue warp stores its own 32 rows, no group
  // barrier) for dense / gather rows.  Conv tiles keep one 128-row box per
  // group: per-warp 4-D boxes measured slower there (halo 3x3 at 56^2:
  // 135 vs 129 us; tools/op_times.py with MS_NO_WARP_STORE=1 as the A/B).
  // The conv coordinates of the per-warp path are kept for the A/B.
  static const bool direct = getenv("MS_DIRECT_STORE") != nullptr;
  p.direct_store = (direct && conv) ? 1 : 0;
  static const bool no_warp_store = getenv("MS_NO_WARP_STORE") != nullptr;
  static const bool conv_warp_store = getenv("MS_CONV_WARP_STORE") != nullptr;
  p.warp_store = (!no_warp_store && (!conv || (conv_warp_store && p.bn == 1 && (p.bw % 32 == 0 || 32 % p.bw == 0) &&
                                               (p.bh * p.bw) % 32 == 0)))
                     ? 1
                     : 0;
  for (int g = 0; g < p.nseg; ++g) {
    const Seg& S = p.seg[g];
    const int w = S.n_end - S.n_begin;
    if (w <= 0 || (S.col0 * 2) % 16 != 0 || (S.ldd * 2) % 16 != 0)
      return set_error(MS_ERR_INVALID, "output segment must be 16-byte aligned (col0, ldd multiples of 8)");
    void* base = reinterpret_cast<__nv_bfloat16*>(S.ptr) + S.col0;
    cuuint32_t es[4] = {1, 1, 1, 1};
    int rc;
    if (conv) {
      cuuint64_t dims[4] = {(cuuint64_t)w, (cuuint64_t)p.OW, (cuuint64_t)p.OH, (cuuint64_t)p.n_img};
      cuuint64_t st[3] = {(cuuint64_t)S.ldd * 2, (cuuint64_t)S.ldd * 2 * p.OW, (cuuint64_t)S.ldd * 2 * p.OW * p.OH};
      cuuint32_t box[4] = {32, (cuuint32_t)p.bw, (cuuint32_t)p.bh, (cuuint32_t)p.bn};
      if (p.warp_store) {
        box[1] = (cuuint32_t)(p.bw >= 32 ? 32 : p.bw);
        box[2] = (cuuint32_t)(p.bw >= 32 ? 1 : 32 / p.bw);
      }
      rc = encode_map(&P->tmD.m[g], 4, base, dims, st, box, es, CU_TENSOR_MAP_SWIZZLE_64B);
    } else {
      cuuint64_t dims[2] = {(cuuint64_t)w, (cuuint64_t)p.M};
      cuuint64_t st[1] = {(cuuint64_t)S.ldd * 2};
      cuuint32_t box[2] = {32, (cuuint32_t)(p.warp_store ? 32 : kBM)};
      rc = encode_map(&P->tmD.m[g], 2, base, dims, st, box, es, CU_TENSOR_MAP_SWIZZLE_64B);
    }
    if (rc) return rc;
  }
  p.tma_store = 1;
  return MS_OK;
}

static void set_segments(GemmParams& p, int nseg, const MsSegment* segs, void* D, long long ldd, int col0) {
  if (nseg <= 0 || segs == nullptr) {
    p.nseg = 1;
    p.seg[0] = Seg{0, p.N, D, ldd, col0, 0};
    return;
  }
  p.nseg = nseg;
  for (int i = 0; i < nseg && i < 4; ++i)
    p.seg[i] = Seg{segs[i].n_begin, segs[i].n_end, segs[i].ptr, segs[i].ldd, segs[i].col0, segs[i].flags};
}

static int launch_plan(const GemmPlan* P, cudaStream_t stream) {
  const GemmParams& p = P->p;
  if (p.mode == MODE_CONV_POOL) return launch_conv_pool(P, stream);
  if (p.mode == MODE_FUSED_HEAD) return launch_fused_head(P, stream);
  if (p.mode == MODE_HEAD_GEMV) return launch_head_gemv(P, stream);
  if (p.mode == MODE_STEM_POOL) {
    static int stem_attr = 0;
    if (!stem_attr) {
      cudaFuncSetAttribute(stem_pool_kernel<true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      cudaFuncSetAttribute(stem_pool_kernel<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      cudaFuncSetAttribute(stem_pool_kernel<true, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      stem_attr = 1;
    }
    if (p.planes == 3)
      launch_k(stem_pool_kernel<true, 3>, dim3(P->grid_x), dim3(kStemThreads), P->smem_bytes, stream, 1, p);
    else if (p.OW <= 112)
      launch_k(stem_pool_kernel<true, 1>, dim3(P->grid_x), dim3(kStemThreads), P->smem_bytes, stream, 1, p);
    else
      launch_k(stem_pool_kernel<false, 1>, dim3(P->grid_x), dim3(kStemThreads), P->smem_bytes, stream, 1, p);
    return check_launch("stem_pool_kernel");
  }
  GemmKernelFn kern = gemm_kernel_for(p);
  if (kern == nullptr) return set_error(MS_ERR_INVALID, "no GEMM kernel for this plan (mode/epilogue)");
  static bool attr_done[64] = {};
  static GemmKernelFn attr_fn[64] = {};
  {  // opt every instantiation into 227 KB of dynamic shared memory once
    int slot = 0;
    while (slot < 64 && attr_fn[slot] != nullptr && attr_fn[slot] != kern) ++slot;
    if (slot < 64 && !attr_done[slot]) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      attr_fn[slot] = kern;
      attr_done[slot] = true;
    }
  }
  launch_k(kern, dim3(P->grid_x, P->grid_y), dim3(kThreads), P->smem_bytes, stream, p.pair ? 2 : 1, P->tmA, P->tmB, p,
           P->tmD);
  int rc = check_launch("gemm_tc_kernel");
  if (rc || p.ksplit <= 1) return rc;
  const long long work = (long long)p.M * ((p.N + 3) / 4);
  long long blocks = (work + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  launch_k(splitk_finalize_kernel, dim3((unsigned)blocks), dim3(256), 0, stream, 1, p);
  return check_launch("splitk_finalize_kernel");
}

}  // namespace mosel

using namespace mosel;

static_assert(sizeof(GemmPlan) <= MS_GEMM_PLAN_BYTES, "MS_GEMM_PLAN_BYTES too small");

extern "C" {

int ms_gemm_plan_dense(void* plan, const void* A, int M, int K, long long lda, const void* W, int N, int K_pad,
                       int BN, const float* bias, int relu, int out_fp32, void* D, long long ldd, int col0,
                       int nseg, const MsSegment* segs) {
  if (plan == nullptr || A == nullptr || W == nullptr) return set_error(MS_ERR_INVALID, "null pointer");
  if (M <= 0 || N <= 0 || K <= 0 || K > K_pad) return set_error(MS_ERR_INVALID, "bad dense GEMM shape");
  if ((lda * 2) % 16 != 0) return set_error(MS_ERR_INVALID, "lda*2 must be a multiple of 16");
  GemmPlan* P = reinterpret_cast<GemmPlan*>(plan);
  memset(P, 0, sizeof(GemmPlan));
  GemmParams& p = P->p;
  p.mode = MODE_DENSE;
  p.M = M;
  p.N = N;
  p.bias = bias;
  p.relu = relu;
  p.out_fp32 = out_fp32;
  p.a_bytes = kABytes;
  set_segments(p, nseg, segs, D, ldd, col0);
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)M};
  cuuint64_t strides[1] = {(cuuint64_t)lda * 2};
  cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)kBM};
  cuuint32_t es[2] = {1, 1};
  int rc = encode_map(&P->tmA, 2, A, dims, strides, box, es);
  if (rc) return rc;
  if (int rc_store = encode_store_maps(P)) return rc_store;
  return finish_plan(P, W, K_pad, N, BN, K_pad / kBK, (M + kBM - 1) / kBM);
}

int ms_gemm_plan_conv(void* plan, const void* X, int n_img, int H, int W_in, int C, long long c_stride, int KH,
                      int KW, int stride, int pad, const void* Wt, int Cout, int BN, const float* bias, int relu,
                      void* D, long long ldd, int col0, int nseg, const MsSegment* segs, int bn, int bh, int bw) {
  if (plan == nullptr || X == nullptr || Wt == nullptr) return set_error(MS_ERR_INVALID, "null pointer");
  if (stride < 1 || stride > 2 || bn * bh * bw > kBM || bn < 1 || bh < 1 || bw < 1)
    return set_error(MS_ERR_INVALID, "bad conv tile / stride");
  if ((c_stride * 2) % 16 != 0 && C != 4 && C != 12)
    return set_error(MS_ERR_INVALID, "channel stride*2 must be a multiple of 16");
  const int OH = (H + 2 * pad - KH) / stride + 1;
  const int OW = (W_in + 2 * pad - KW) / stride + 1;
  GemmPlan* P = reinterpret_cast<GemmPlan*>(plan);
  memset(P, 0, sizeof(GemmPlan));
  GemmParams& p = P->p;
  p.mode = MODE_CONV;
  p.N = Cout;
  p.bias = bias;
  p.relu = relu;
  p.n_img = n_img;
  p.OH = OH;
  p.OW = OW;
  p.stride = stride;
  p.pad = pad;
  p.KW = KW;
  p.cchunks = (C + kBK - 1) / kBK;
  p.bn = bn;
  p.bh = bh;
  p.bw = bw;
  p.tiles_w = (OW + bw - 1) / bw;
  p.tiles_h = (OH + bh - 1) / bh;
  p.a_bytes = bn * bh * bw * kBK * 2;
  p.M = n_img * OH * OW;
  set_segments(p, nseg, segs, D, ldd, col0);
  cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W_in, (cuuint64_t)H, (cuuint64_t)n_img};
  cuuint64_t strides[3] = {(cuuint64_t)c_stride * 2, (cuuint64_t)c_stride * 2 * W_in,
                           (cuuint64_t)c_stride * 2 * W_in * H};
  cuuint32_t es[4] = {1, (cuuint32_t)stride, (cuuint32_t)stride, 1};
  int num_kb;
  if (C == 12) {
    // X is [n_img, H + 2*pad, W_in + 2*pad, 12]: rows and columns pre-padded
    if (stride != 2 || KW > 8 || KH > 8) return set_error(MS_ERR_INVALID, "12-channel conv needs stride 2, KH/KW <= 8");
    p.mode = MODE_CONV_C12;
    p.a_bytes = bn * bh * bw * 128;
    p.smallc_halves = 3 * KH;            // 32-element parts of the filter-row windows
    num_kb = (3 * KH + 1) / 2;
    const long long wp = W_in + 2LL * pad, hp = H + 2LL * pad;
    const long long pitch = wp * 12 * 2;
    cuuint64_t d4[4] = {96, (cuuint64_t)OW, (cuuint64_t)hp, (cuuint64_t)n_img};
    cuuint64_t s4[3] = {48, (cuuint64_t)pitch, (cuuint64_t)(pitch * hp)};
    cuuint32_t b4[4] = {32, (cuuint32_t)bw, (cuuint32_t)(bh * 2), (cuuint32_t)bn};
    cuuint32_t e4[4] = {1, 1, 2, 1};
    int rc = encode_map(&P->tmA, 4, X, d4, s4, b4, e4, CU_TENSOR_MAP_SWIZZLE_64B);
    if (rc) return rc;
  } else if (C == 4) {
    // X is [n_img, H + 2*pad, W_in + 2*pad, 4]: rows and columns pre-padded
    if (stride != 2 || KW > 8 || KH > 8) return set_error(MS_ERR_INVALID, "4-channel conv needs stride 2, KH/KW <= 8");
    p.mode = MODE_CONV_C4;
    p.a_bytes = bn * bh * bw * 128;
    num_kb = (KH + 1) / 2;
    const long long wp = W_in + 2LL * pad, hp = H + 2LL * pad;
    const long long pitch = wp * 4 * 2;
    cuuint64_t d4[4] = {32, (cuuint64_t)OW, (cuuint64_t)hp, (cuuint64_t)n_img};
    cuuint64_t s4[3] = {16, (cuuint64_t)pitch, (cuuint64_t)(pitch * hp)};
    cuuint32_t b4[4] = {32, (cuuint32_t)bw, (cuuint32_t)(bh * 2), (cuuint32_t)bn};
    cuuint32_t e4[4] = {1, 1, 2, 1};
    int rc = encode_map(&P->tmA, 4, X, d4, s4, b4, e4, CU_TENSOR_MAP_SWIZZLE_64B);
    if (rc) return rc;
  } else if (C < kBK) {
    // X is [n_img, H, W_in + 2*pad, C] (W pre-padded with zeros)
    if (C != 8 && C != 16) return set_error(MS_ERR_INVALID, "small-channel conv needs C == 8 or 16 (padded)");
    if (KW > 8) return set_error(MS_ERR_INVALID, "small-channel conv supports KW <= 8");
    p.mode = MODE_CONV_SMALLC;
    p.smallc_jpb = 64 / C;          // window pixels per 128-B row
    p.smallc_halves = 8 / p.smallc_jpb;
    p.a_bytes = bn * bh * bw * 128;
    num_kb = KH * p.smallc_halves;
    const long long wp = W_in + 2LL * pad;
    // dim0 = the contiguous 8-pixel window (8*C elements) starting at padded
    // column ow*stride; dim1 = output column, stride `stride` pixels (the
    // windows overlap); dim2 = input row (element stride = conv stride)
    cuuint64_t d5[4] = {(cuuint64_t)(8 * C), (cuuint64_t)OW, (cuuint64_t)H, (cuuint64_t)n_img};
    cuuint64_t s5[3] = {(cuuint64_t)C * 2 * stride, (cuuint64_t)(wp * C * 2), (cuuint64_t)(wp * C * 2 * H)};
    cuuint32_t b5[4] = {(cuuint32_t)kBK, (cuuint32_t)bw, (cuuint32_t)(bh * stride), (cuuint32_t)bn};
    cuuint32_t e5[4] = {1, 1, (cuuint32_t)stride, 1};
    int rc = encode_map(&P->tmA, 4, X, d5, s5, b5, e5);
    if (rc) return rc;
  } else {
    cuuint32_t box[4] = {(cuuint32_t)kBK, (cuuint32_t)(bw * stride), (cuuint32_t)(bh * stride), (cuuint32_t)bn};
    int rc = encode_map(&P->tmA, 4, X, dims, strides, box, es);
    if (rc) return rc;
    num_kb = KH * KW * p.cchunks;
  }
  const int tiles_n = (n_img + bn - 1) / bn;
  if (int rc_store = encode_store_maps(P)) return rc_store;
  return finish_plan(P, Wt, num_kb * kBK, Cout, BN, num_kb, tiles_n * p.tiles_h * p.tiles_w);
}

int ms_gemm_plan_conv_k32(void* plan, const void* X, int n_img, int H, int W_in, int C, long long c_stride, int KH,
                          int KW, int stride, int pad, const void* Wt, int Cout, int BN, const float* bias, int relu,
                          void* D, long long ldd, int col0, int nseg, const MsSegment* segs, int bn, int bh, int bw) {
  if (C % 32 != 0 || C % 64 == 0 || KH * KW != 9)
    return set_error(MS_ERR_INVALID, "k32 conv: 3x3 with input channels a multiple of 32 but not of 64");
  int rc = ms_gemm_plan_conv(plan, X, n_img, H, W_in, C, c_stride, KH, KW, stride, pad, Wt, Cout, BN, bias, relu, D,
                             ldd, col0, nseg, segs, bn, bh, bw);
  if (rc) return rc;
  GemmPlan* P = reinterpret_cast<GemmPlan*>(plan);
  GemmParams& p = P->p;
  if (p.mode != MODE_CONV) return set_error(MS_ERR_INVALID, "k32 conv: unexpected mode");
  cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W_in, (cuuint64_t)H, (cuuint64_t)n_img};
  cuuint64_t strides[3] = {(cuuint64_t)c_stride * 2, (cuuint64_t)c_stride * 2 * W_in,
                           (cuuint64_t)c_stride * 2 * W_in * H};
  cuuint32_t box[4] = {32, (cuuint32_t)(bw * stride), (cuuint32_t)(bh * stride), (cuuint32_t)bn};
  cuuint32_t es[4] = {1, (cuuint32_t)stride, (cuuint32_t)stride, 1};
  rc = encode_map(&P->tmA, 4, X, dims, strides, box, es, CU_TENSOR_MAP_SWIZZLE_64B);
  if (rc) return rc;
  p.mode = MODE_CONV_K32;
  p.cchunks = C / 32;  // 32-channel parts per tap
  p.num_kb = (9 * p.cchunks + 1) / 2;
  p.kb_per = p.num_kb;
  // weights [Cout, num_kb * 64]: K = tap * C + c, zero padded to whole blocks
  cuuint64_t wd[2] = {(cuuint64_t)(p.num_kb * kBK), (cuuint64_t)Cout};
  cuuint64_t ws[1] = {(cuuint64_t)p.num_kb * kBK * 2};
  cuuint32_t wb[2] = {(cuuint32_t)kBK, (cuuint32_t)p.BN};
  cuuint32_t we[2] = {1, 1};
  rc = encode_map(&P->tmB, 2, Wt, wd, ws, wb, we);
  if (rc) return rc;
  P->w_kpad = p.num_kb * kBK;
  if (p.stages > p.num_kb) p.stages = p.num_kb < 2 ? 2 : p.num_kb;
  return MS_OK;
}

int ms_gemm_plan_conv_halo(void* plan, const void* X, int n_img, int H, int W_in, int C, long long c_stride,
                           const void* Wt, int Cout, int BN, const float* bias, int relu, void* D, long long ldd,
                           int col0, int nseg, const MsSegment* segs) {
  if (W_in < 14 || C < 64) return set_error(MS_ERR_INVALID, "halo conv: width >= 14 and >= 64 input channels");
  const int P = ((W_in + 2) + 7) / 8 * 8;
  if (128 % P != 0) return set_error(MS_ERR_INVALID, "halo conv: padded row width must divide 128 (W <= 62)");
  const int bh = 128 / P;
  // a 3x3/1/1 conv plan with (1 image x bh rows x P columns) output tiles; then
  // the A map becomes one (bh + 2) x P halo box per 64-channel chunk
  int rc = ms_gemm_plan_conv(plan, X, n_img, H, W_in, C, c_stride, 3, 3, 1, 1, Wt, Cout, BN, bias, relu, D, ldd,
                             col0, nseg, segs, 1, bh, P);
  if (rc) return rc;
  GemmPlan* Pl = reinterpret_cast<GemmPlan*>(plan);
  GemmParams& p = Pl->p;
  if (p.mode != MODE_CONV || p.tiles_w != 1) return set_error(MS_ERR_INVALID, "halo conv: unexpected tiling");
  cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W_in, (cuuint64_t)H, (cuuint64_t)n_img};
  cuuint64_t strides[3] = {(cuuint64_t)c_stride * 2, (cuuint64_t)c_stride * 2 * W_in,
                           (cuuint64_t)c_stride * 2 * W_in * H};
  cuuint32_t box[4] = {(cuuint32_t)kBK, (cuuint32_t)P, (cuuint32_t)(bh + 2), 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  rc = encode_map(&Pl->tmA, 4, X, dims, strides, box, es);
  if (rc) return rc;
  p.mode = MODE_CONV_HALO;
  p.occ2 = 0;  // halo plans keep one CTA per SM (resident weights / halo ring)
  p.single_acc = 0;
  {
    int tc = 32;
    while (tc < p.BN) tc <<= 1;
    Pl->tmem_cols = 2 * tc;
    const int tiles = p.m_tiles * ((p.N + p.BN - 1) / p.BN);
    Pl->grid_x = tiles < sm_count() ? tiles : sm_count();
  }
  p.a_bytes = kBK * P * (bh + 2) * 2;
  // + 2 rows: the last tap's shifted view of the last M rows reads past the halo
  p.halo_slot = ((p.a_bytes + 2 * 128) + 1023) / 1024 * 1024;
  const int bias_bytes = ((p.N + 31) / 32) * 32 * 4;
  const int room = 226 * 1024 - 1024 - 288 - 2 * p.halo_slot - p.stage_bytes - bias_bytes;
  // an N tile whose 9 x cchunks weight blocks fit stays resident; each CTA
  // then serves one N tile (grid rounded to a multiple of the N tiles).
  // Splitting N to make the weights fit measured slower (halo reloads per N
  // tile + narrower MMAs; profiles/r01_halo_bench.txt): one N tile only.
  const int n_tiles = (p.N + p.BN - 1) / p.BN;
  p.b_resident = (n_tiles == 1 && 9 * p.cchunks * p.b_bytes <= room) ? 1 : 0;
  int stages = p.b_resident ? 9 * p.cchunks : room / p.b_bytes;
  if (!p.b_resident && stages > kMaxHaloStages) stages = kMaxHaloStages;  // weights-only stages are small
  if (p.b_resident) {
    const int tiles = p.m_tiles * n_tiles;
    int g = tiles < sm_count() ? tiles : sm_count();
    g = (g / n_tiles) * n_tiles;
    Pl->grid_x = g < n_tiles ? n_tiles : g;
  }
  if (stages < 2) return set_error(MS_ERR_INVALID, "halo conv: weights tile does not fit");
  p.stages = stages;
  Pl->smem_bytes = 1024 + 2 * p.halo_slot + stages * p.b_bytes + p.stage_bytes + (2 * stages + 8) * 8 + 16 + bias_bytes;
  return MS_OK;
}

int ms_gemm_plan_gather(void* plan, const void* const* feat, const int32_t* inv, int inv_ld, int n_mod,
                        int feat_dim, int M, const void* W, int N, int BN, const float* bias, int relu,
                        int out_fp32, void* D, long long ldd, int col0) {
  if (plan == nullptr || feat == nullptr || inv == nullptr || W == nullptr)
    return set_error(MS_ERR_INVALID, "null pointer");
  if (n_mod < 1 || n_mod > 4 || feat_dim % kBK != 0 || M <= 0)
    return set_error(MS_ERR_INVALID, "gather GEMM needs 1..4 modalities and feat_dim % 64 == 0");
  GemmPlan* P = reinterpret_cast<GemmPlan*>(plan);
  memset(P, 0, sizeof(GemmPlan));
  GemmParams& p = P->p;
  p.mode = MODE_GATHER;
  p.M = M;
  p.N = N;
  p.bias = bias;
  p.relu = relu;
  p.out_fp32 = out_fp32;
  p.inv = inv;
  p.inv_ld = inv_ld;
  p.n_mod = n_mod;
  p.feat_dim = feat_dim;
  for (int k = 0; k < n_mod; ++k) p.feat[k] = reinterpret_cast<const __nv_bfloat16*>(feat[k]);
  for (int k = n_mod; k < 4; ++k) p.feat[k] = p.feat[0];
  set_segments(p, 0, nullptr, D, ldd, col0);
  const int K = n_mod * feat_dim;
  if (int rc_store = encode_store_maps(P)) return rc_store;
  return finish_plan(P, W, K, N, BN, K / kBK, (M + kBM - 1) / kBM);
}

int ms_gemm_plan_set_residual(void* plan, const void* residual, long long res_ld) {
  GemmPlan* P = reinterpret_cast<GemmPlan*>(plan);
  if (P == nullptr) return set_error(MS_ERR_INVALID, "null plan");
  if (P->p.out_fp32 || P->p.nseg > 1 || (res_ld * 2) % 16 != 0)
    return set_error(MS_ERR_INVALID, "residual needs a bf16 single-segment output and res_ld*2 % 16 == 0");
  P->p.residual = reinterpret_cast<const __nv_bfloat16*>(residual);
  P->p.res_ld = res_ld;
  return MS_OK;
}

int ms_gemm_plan_set_splitk(void* plan, int ksplit, float* ws, long long ws_ld) {
  GemmPlan* P = reinterpret_cast<GemmPlan*>(plan);
  if (P == nullptr) return set_error(MS_ERR_INVALID, "null plan");
  GemmParams& p = P->p;
  if (ksplit < 1) return set_error(MS_ERR_INVALID, "ksplit must be >= 1");
  if (ksplit > 1) {
    if (p.mode == MODE_CONV_SMALLC || p.pair || p.nseg > 1 || ws == nullptr ||
        ws_ld % 4 != 0 || ws_ld < p.N)
      return set_error(MS_ERR_INVALID,
                       "split-K needs a dense/gather/conv single-segment plan and ws[ksplit, M, ws_ld>=N, %4]");
  }
  const int kb_per = (p.num_kb + ksplit - 1) / ksplit;
  p.ksplit = (p.num_kb + kb_per - 1) / kb_per;  // no empty K parts
  p.kb_per = kb_per;
  p.ws = ws;
  p.ws_ld = ws_ld;
  if (p.ksplit > 1) {
    p.tma_store = 0;  // partial sums go to the fp32 workspace (layout unchanged)
    p.occ2 = 0;
    p.single_acc = 0;
  }
  // (grid recomputed below for the split tiles)
  const int tiles = p.m_tiles * ((p.N + p.BN - 1) / p.BN) * p.ksplit;
  P->grid_x = tiles < sm_count() ? tiles : sm_count();
  return MS_OK;
}

int ms_gemm_plan_set_pair(void* plan, int enable) {
  GemmPlan* P = reinterpret_cast<GemmPlan*>(plan);
  if (P == nullptr) return set_error(MS_ERR_INVALID, "null plan");
  GemmParams& p = P->p;
  if (!enable || p.pair) return MS_OK;
  if ((p.mode != MODE_DENSE && p.mode != MODE_CONV && p.mode != MODE_CONV_K32 && p.mode != MODE_CONV_HALO) ||
      p.ksplit > 1 || p.out_fp32 || !p.tma_store || p.BN % 32 != 0)
    return set_error(MS_ERR_INVALID, "CTA-pair mode needs a dense/conv/k32/halo bf16 plan without split-K");
  // the weight box becomes BN/2 rows per CTA
  cuuint64_t dims[2] = {(cuuint64_t)P->w_kpad, (cuuint64_t)P->w_rows};
  cuuint64_t strides[1] = {(cuuint64_t)P->w_kpad * 2};
  cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)(p.BN / 2)};
  cuuint32_t es[2] = {1, 1};
  int rc = encode_map(&P->tmB, 2, P->w_ptr, dims, strides, box, es);
  if (rc) return rc;
  p.pair = 1;
  p.occ2 = 0;
  p.single_acc = 0;
  p.b_bytes = (p.BN / 2) * kBK * 2;
  const int bias_bytes = ((p.N + 31) / 32) * 32 * 4;
  const int n_tiles = (p.N + p.BN - 1) / p.BN;
  const int pair_tiles = ((p.m_tiles + 1) / 2) * n_tiles;
  int clusters = pair_tiles < sm_count() / 2 ? pair_tiles : sm_count() / 2;
  if (p.mode == MODE_CONV_HALO) {
    const int room = 226 * 1024 - 1024 - 288 - 2 * p.halo_slot - p.stage_bytes - bias_bytes;
    // half of the weights per CTA: layers whose full tile did not fit can now stay resident
    // (with several N tiles the grid is a multiple of n_tiles, so each pair keeps one N tile)
    p.b_resident = (9 * p.cchunks * p.b_bytes <= room) ? 1 : 0;
    int stages = p.b_resident ? 9 * p.cchunks : room / p.b_bytes;
    if (!p.b_resident && stages > kMaxHaloStages) stages = kMaxHaloStages;
    if (stages < 2) return set_error(MS_ERR_INVALID, "halo pair: weights tile does not fit");
    p.stages = stages;
    P->smem_bytes = 1024 + 2 * p.halo_slot + stages * p.b_bytes + p.stage_bytes + (2 * stages + 8) * 8 + 16 + bias_bytes;
    if (p.b_resident) clusters = clusters / n_tiles * n_tiles < n_tiles ? n_tiles : clusters / n_tiles * n_tiles;
  } else {
    const int per_stage = kABytes + p.b_bytes;
    int stages = (226 * 1024 - 1024 - 288 - p.stage_bytes - bias_bytes) / per_stage;
    if (stages > max_stages()) stages = max_stages();
    if (stages > p.num_kb) stages = p.num_kb < 2 ? 2 : p.num_kb;
    p.stages = stages;
    P->smem_bytes = 1024 + stages * per_stage + p.stage_bytes + (2 * stages + 8) * 8 + 16 + bias_bytes;
  }
  if (P->smem_bytes > 227 * 1024) return set_error(MS_ERR_INVALID, "pair plan exceeds 227 KB shared memory");
  P->grid_x = 2 * clusters;
  P->grid_y = 1;
  return MS_OK;
}

int ms_set_occ2_grid(int mode) {
  const int prev = g_occ2_grid;
  g_occ2_grid = mode;
  return prev;
}

int ms_gemm_plan_set_trace(void* plan, unsigned long long* buf) {
  GemmPlan* P = reinterpret_cast<GemmPlan*>(plan);
  if (P == nullptr) return set_error(MS_ERR_INVALID, "null plan");
  P->p.trace = buf;
  return MS_OK;
}

int ms_gemm_plan_debug(void* plan, int flags) {
  GemmPlan* P = reinterpret_cast<GemmPlan*>(plan);
  if (P == nullptr) return set_error(MS_ERR_INVALID, "null plan");
  P->p.debug_flags = flags;
  return MS_OK;
}

// 7x7/2 conv over pre-padded 4-channel pixels + bias + ReLU + 3x3/2 ceil-mode
// max pool in one kernel (MODE_STEM_POOL).  X: [n_img, H + 2*pad, W + 2*pad, 4]
// bf16; Wt: [64, 256] bf16 in the C4 packing (K = (kh, 8 px, 4 ch)); Y: pooled
// [n_img, PH, PW] rows of ldy elements, 64 channels at y_col0.
int ms_gemm_plan_stem_pool(void* plan, const void* X, int n_img, int H, int W_in, int KH, int pad, int planes,
                           long long plane_stride, const void* Wt, const float* bias, void* Y, long long ldy,
                           int y_col0) {
  if (plan == nullptr || X == nullptr || Wt == nullptr || Y == nullptr) return set_error(MS_ERR_INVALID, "null pointer");
  if (KH != kStemKH || n_img < 1) return set_error(MS_ERR_INVALID, "stem conv needs a 7x7 filter, n_img >= 1");
  const int OH = (H + 2 * pad - KH) / 2 + 1, OW = (W_in + 2 * pad - KH) / 2 + 1;
  if (OW > kBM || OH < 3 || OW < 3) return set_error(MS_ERR_INVALID, "stem conv needs 3 <= output width <= 128");
  if (H + 2 * pad < 2 * OH + 5)  // the last conv row's 7 input rows lie inside the padded frame
    return set_error(MS_ERR_INVALID, "stem conv: padded frame too short");
  const long long pitch = (long long)(W_in + 2 * pad) * 4 * 2;
  if (pitch % 16 != 0) return set_error(MS_ERR_INVALID, "padded stem row must be a multiple of 16 bytes");
  if ((reinterpret_cast<uintptr_t>(X) & 15) != 0 || (reinterpret_cast<uintptr_t>(Y) & 15) != 0 || (ldy % 8) != 0 ||
      (y_col0 % 8) != 0)
    return set_error(MS_ERR_INVALID, "stem input and output rows must be 16-B aligned");
  // ceil-mode 3x3/2 pool without padding: the last window starts inside the map
  const int PH = (OH - 3 + 1) / 2 + 1, PW = (OW - 3 + 1) / 2 + 1;
  GemmPlan* P = reinterpret_cast<GemmPlan*>(plan);
  memset(P, 0, sizeof(GemmPlan));
  GemmParams& p = P->p;
  p.mode = MODE_STEM_POOL;
  p.N = 64;
  p.BN = 64;
  p.bias = bias;
  p.relu = MS_ACT_RELU;
  p.n_img = n_img;
  p.OH = OH;
  p.OW = OW;
  p.stride = 2;
  p.pad = pad;
  p.KW = KH;
  p.M = n_img * OH * OW;
  p.xraw = reinterpret_cast<const uint8_t*>(X);
  p.x_pitch = pitch;
  p.Hp = H + 2 * pad;
  p.PH = PH;
  p.PW = PW;
  p.units = n_img * PH;
  if (planes != 1 && planes != 3) return set_error(MS_ERR_INVALID, "stem conv: planes must be 1 or 3");
  if (planes == 3 && (OW > 112 || plane_stride <= 0 || (plane_stride * 2) % 16 != 0))
    return set_error(MS_ERR_INVALID, "stem conv: 3 planes need output width <= 112 and a 16-B plane stride");
  p.planes = planes;
  p.x_plane = plane_stride * 2;
  p.a_bytes = (int)(kStemMaxRows * pitch);       // a CLOSE tile's input rows (per plane)
  p.plane_bytes = (p.a_bytes + 127) / 128 * 128;
  p.b_bytes = planes * p.plane_bytes;            // stage stride
  p.nseg = 1;
  p.seg[0] = Seg{0, 64, Y, ldy, y_col0, 0};
  if ((reinterpret_cast<uintptr_t>(Wt) & 15) != 0) return set_error(MS_ERR_INVALID, "stem weights must be 16-B aligned");
  p.wraw = reinterpret_cast<const uint8_t*>(Wt);
  P->w_ptr = Wt;
  const bool overlap = OW <= 112;
  const int w_bytes = planes == 1 ? kStemWBytes : kStemKH * planes * kStemWBlk;
  const int fixed = 1024 + w_bytes + 256 + (overlap ? 0 : kStemRowBuf) + 1024;
  int stages = (226 * 1024 - fixed) / p.b_bytes;
  if (stages > 8) stages = 8;
  if (stages < 2) return set_error(MS_ERR_INVALID, "stem rows too wide for shared memory");
  p.stages = stages;
  P->smem_bytes = fixed + stages * p.b_bytes;
  P->grid_x = p.units < sm_count() ? p.units : sm_count();
  P->grid_y = 1;
  P->tmem_cols = 512;
  return MS_OK;
}

int ms_gemm_plan_stem_set_reduce(void* plan, const void* Wred, const float* bias, void* Y, long long ldy, int y_col0) {
  GemmPlan* P = reinterpret_cast<GemmPlan*>(plan);
  if (P == nullptr || Wred == nullptr || Y == nullptr) return set_error(MS_ERR_INVALID, "null pointer");
  GemmParams& p = P->p;
  if (p.mode != MODE_STEM_POOL || p.OW > 112)
    return set_error(MS_ERR_INVALID, "stem reduce: needs a stem_pool plan with output width <= 112");
  if ((reinterpret_cast<uintptr_t>(Wred) & 15) != 0 || (reinterpret_cast<uintptr_t>(Y) & 15) != 0 || ldy % 8 != 0 ||
      y_col0 % 8 != 0)
    return set_error(MS_ERR_INVALID, "stem reduce: weights and output rows must be 16-B aligned");
  p.red_w = reinterpret_cast<const uint8_t*>(Wred);
  p.red_bias = bias;
  p.seg[1] = Seg{0, 64, Y, ldy, y_col0, 0};
  // shared memory: + two pooled-row A tiles + the 1x1 weights (1 KB aligned) + barriers
  const int w_bytes = p.planes == 1 ? kStemWBytes : kStemKH * p.planes * kStemWBlk;
  const int extra = 1024 + 2 * kStemRedA + kStemRedW + 6 * 8 + 256;
  int stages = p.stages;
  while (stages > 1 && 1024 + w_bytes + 256 + stages * p.b_bytes + extra + (2 * stages + 1 + 2 * kStemSlots) * 8 +
                            16 + 512 > 227 * 1024)
    --stages;
  const int bytes = 1024 + w_bytes + 256 + stages * p.b_bytes + extra + (2 * stages + 1 + 2 * kStemSlots) * 8 + 16 + 512;
  if (stages < 2 || bytes > 227 * 1024) return set_error(MS_ERR_INVALID, "stem reduce: does not fit in shared memory");
  p.stages = stages;
  P->smem_bytes = bytes;
  return MS_OK;
}

int ms_gemm_run(const void* plan, void* stream) {
  if (plan == nullptr) return set_error(MS_ERR_INVALID, "null plan");
  return launch_plan(reinterpret_cast<const GemmPlan*>(plan), reinterpret_cast<cudaStream_t>(stream));
}

int ms_gemm_plan_info(const void* plan, int* grid_x, int* grid_y, int* stages, int* smem_bytes) {
  const GemmPlan* P = reinterpret_cast<const GemmPlan*>(plan);
  if (P == nullptr) return set_error(MS_ERR_INVALID, "null plan");
  if (grid_x) *grid_x = P->grid_x;
  if (grid_y) *grid_y = P->grid_y;
  if (stages) *stages = P->p.stages;
  if (smem_bytes) *smem_bytes = P->smem_bytes;
  return MS_OK;
}

}  // extern "C"
