// Fused late-fusion head: masked concat -> FC1 (K*F -> 512) + ReLU -> FC2
// (512 -> classes) -> fp32 logits, in ONE launch of 8-CTA clusters.
//
// Reference: the fusion MLP applied after the per-modality encoders
// (reference: profile.py:157-159 drops absent modalities; the
// oracle/forward.py fusion_forward restatement is the checker).  The unfused
// device path is three launches (gather-concat GEMM, FC2 split-K GEMM, the
// split-K finalize) with h and the partial logits round-tripping through HBM.
//
// One cluster of CL = 8 CTAs per 128-request tile.  Phase 1: CTA r multiplies
// its K slice (K / 8 columns of the concatenated features, gathered straight
// from the compacted per-modality rows through inv -- absent modalities are
// zero rows) by the matching W1 columns: a [128 x 512] fp32 partial in TMEM
// (two N = 256 MMAs per K step).  Phase 2: reduce-scatter over distributed
// shared memory -- CTA o owns hidden columns [64 o, 64 o + 64).  Every CTA
// stages its slices for the other owners from TMEM into local shared memory
// and ONE thread moves each with a bulk copy (cp.async.bulk shared::cta ->
// shared::cluster, completing on the owner's mbarrier): DSMEM throughput is
// message bound, so per-thread st.shared::cluster was 5x slower.  Owners add
// the slices in a fixed source order (deterministic, no atomics).  Only the
// rows holding requests move (vpad = valid rows rounded up to 8).  Phase 3:
// the owner applies bias + ReLU, rounds h to bf16 (the unfused path's
// rounding point) into its 64-column chunk of a [128 x 512] SW128 K-major h
// tile and bulk-copies that chunk into the 7 other CTAs' h tiles (all-gather,
// bf16: half the bytes of a second fp32 reduce-scatter).  Phase 4: CTA r
// computes logits columns [64 r, 64 r + 64) = h . W2[64 r : 64 r + 64]^T over
// the full K = 512 (N = 64 MMAs, W2 rows by TMA), adds b2 and stores the
// valid rows -- every logit has exactly one producer, in K order.
//
// Shared memory (227 KB): a 224 KB window = 2 pipeline stages x (A 16 KB +
// W1 64 KB) during phase 1, then the phase-2 send and receive slots
// ([16 chunks of 4 columns][vpad rows][16 B], so the staging stores are
// conflict free and a slice is one contiguous bulk copy; rounds when 7 + 7
// slots do not fit), then the h tile (128 KB); the W2 slice sits above the
// stages (160 KB) and loads at kernel start when the slots fit below it
// (tiles of <= 40 requests), else right after phase 2.
#include <cstdio>

#include "gemm_plan.h"
#include "ptx.cuh"
#include "runtime.h"

namespace mosel {

namespace {

constexpr int kHdThreads = 256;
constexpr int kHdCL = 8;                       // CTAs per cluster (one 128-request tile)
constexpr int kHdHidden = 512;                 // FC1 outputs (FUSION_HIDDEN)
constexpr int kHdSlice = kHdHidden / kHdCL;    // 64 owned columns per CTA
constexpr int kHdWBytes = kHdHidden * kBK * 2; // one W1 K block: 512 rows x 128 B
constexpr int kHdStage = kABytes + kHdWBytes;  // 80 KB
constexpr int kHdR0 = 2 * kHdStage;            // 160 KB
constexpr int kHdWindow = 224 * 1024;          // phase-2 slot window (stages, then h + W2)
constexpr int kHdHTile = kBM * kHdHidden * 2;  // 128 KB: 8 SW128 chunks of 64 hidden columns
constexpr int kHdHChunk = kBM * 128;           // 16 KB
constexpr int kHdW2Off = kHdR0;                // after the stages: loadable at kernel start
constexpr int kHdW2Chunk = kHdSlice * 128;     // 64 W2 rows x 64 K (bf16) = 8 KB
constexpr int kHdW2Bytes = 8 * kHdW2Chunk;     // 64 KB
constexpr int kHdBarOff = kHdWindow;
constexpr int kHdSmem = 1024 + kHdBarOff + 256 + 2 * kHdSlice * 4;
static_assert(kHdR0 <= kHdWindow && kHdW2Off + kHdW2Bytes <= kHdWindow, "layout");
static_assert(kHdSmem <= 227 * 1024, "fused head exceeds 227 KB");

// one bulk copy from this CTA's shared memory into a peer's, completing
// (complete_tx) on the peer's mbarrier; dst and bar are shared::cluster addresses
__device__ __forceinline__ void bulk_s2s_cluster(uint32_t dst, uint32_t src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "r"(src), "r"(bytes), "r"(bar)
      : "memory");
}

// slots per phase-2 round (send + receive) for vpad live rows
// within a window of `win` bytes
__host__ __device__ constexpr int hd_round_slots(int vpad, int win) {
  return (win / (2 * vpad * 256)) < kHdCL - 1 ? (win / (2 * vpad * 256)) : kHdCL - 1;
}
static_assert(hd_round_slots(128, kHdWindow) >= 3, "at most three rounds");
// W2 early: all phase-2 slots fit below the W2 slice (one round), so W2 loads at kernel start
__host__ __device__ constexpr bool hd_w2_early(int vpad) { return 2 * (kHdCL - 1) * vpad * 256 <= kHdR0; }

// W2 rows [64 r, 64 r + 64) (>= classes: zero fill), one 8 KB box per K chunk
__device__ __forceinline__ void load_w2(uint8_t* w2s, const CUtensorMap* tmW2, uint64_t* w2bar, uint32_t rank) {
  mbar_arrive_expect_tx(w2bar, kHdW2Bytes);
  for (int kc = 0; kc < 8; ++kc)
    tma_load_2d(smem_addr(w2s) + kc * kHdW2Chunk, tmW2, w2bar, kc * kBK, (int)rank * kHdSlice);
}

// Phase 2: on return acc[] = sum over the 8 CTAs of hidden columns
// rank*64 + half*32 + [0, 32) of this thread's row (own partial first, then
// sources rank-1, rank-2, ... mod 8: a fixed order, bitwise reproducible).
__device__ __forceinline__ void reduce_scatter(float (&acc)[32], uint32_t taddr_row, uint8_t* win, uint32_t rank,
                                               int row, int half, bool live, int vpad, int wbytes, uint64_t* rbar) {
  uint32_t v[32];
  if (live) {
    tmem_ld_32x32b_x32(taddr_row + rank * kHdSlice + half * 32, v);
    tmem_wait_ld();
#pragma unroll
    for (int c = 0; c < 32; ++c) acc[c] = __uint_as_float(v[c]);
  }
  const uint32_t plane = (uint32_t)vpad * 16, slot_bytes = plane * 16;
  const int S = hd_round_slots(vpad, wbytes);
  uint8_t* recv = win;                  // slots [0, S)
  uint8_t* send = win + S * slot_bytes; // slots [S, 2S)
#pragma unroll 1
  for (int j0 = 0, rd = 0; j0 < kHdCL - 1; j0 += S, ++rd) {
    const int jn = min(kHdCL - 1, j0 + S);
    if (threadIdx.x == 0) mbar_arrive_expect_tx(&rbar[rd], (jn - j0) * slot_bytes);
    if (live) {
#pragma unroll 1
      for (int j = j0; j < jn; ++j) {
        const uint32_t o = (rank + 1 + j) % kHdCL;
        tmem_ld_32x32b_x32(taddr_row + o * kHdSlice + half * 32, v);
        tmem_wait_ld();
        uint8_t* dst = send + (j - j0) * slot_bytes + row * 16;
        if (row < vpad) {
#pragma unroll
          for (int c = 0; c < 8; ++c)
            *reinterpret_cast<uint4*>(dst + (half * 8 + c) * plane) =
                make_uint4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
        }
      }
    }
    fence_proxy_async_smem();  // generic stores -> bulk-copy (async proxy) reads
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int j = j0; j < jn; ++j) {  // source rank lands in slot j - j0 of owner o
        const uint32_t o = (rank + 1 + j) % kHdCL;
        bulk_s2s_cluster(mapa_shared(smem_addr(recv + (j - j0) * slot_bytes), o),
                         smem_addr(send + (j - j0) * slot_bytes), slot_bytes, mapa_shared(smem_addr(&rbar[rd]), o));
      }
    }
    mbar_wait(&rbar[rd], 0);
    if (live && row < vpad) {
#pragma unroll 1
      for (int j = j0; j < jn; ++j) {  // slot j - j0 holds source rank - 1 - j
        const uint8_t* src = recv + (j - j0) * slot_bytes + row * 16;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float4 f = *reinterpret_cast<const float4*>(src + (half * 8 + c) * plane);
          acc[4 * c] += f.x;
          acc[4 * c + 1] += f.y;
          acc[4 * c + 2] += f.z;
          acc[4 * c + 3] += f.w;
        }
      }
    }
    // every owner has its slices (so every send slot was read) and has read
    // them (receive slots free): the next round / the h all-gather may write
    cluster_sync_all();
  }
}

__global__ void __launch_bounds__(kHdThreads, 1)
    fused_head_kernel(const __grid_constant__ CUtensorMap tmW2, const __grid_constant__ CUtensorMap tmW1,
                      const __grid_constant__ GemmParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
  uint8_t* r0 = smem;               // phase 1 stages | phase 2 slots | h tile
  uint8_t* w2s = smem + kHdW2Off;   // W2 slice (after phase 2)
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kHdBarOff);
  uint64_t* empty = full + 2;
  uint64_t* tfull = empty + 2;  // [0]: FC1 partial done, [1]: FC2 done
  uint64_t* w2bar = tfull + 2;
  uint64_t* hbar = w2bar + 1;   // the 7 peer h chunks arrived
  uint64_t* rbar = hbar + 1;    // phase-2 rounds (<= 3)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rbar + 3);
  float* sb1 = reinterpret_cast<float*>(tmem_slot + 4);  // this CTA's 64 b1 / b2 columns
  float* sb2 = sb1 + kHdSlice;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int m_tile = blockIdx.x / kHdCL;
  const int KB = p.num_kb;  // K blocks per CTA
  const int kb0 = (int)rank * KB;
  const int valid = min(kBM, p.M - m_tile * kBM);
  const int vpad = (valid + 7) / 8 * 8;  // rows moved between CTAs
  const bool w2_early = hd_w2_early(vpad);
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&full[s], 1 + kBM);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&tfull[0], 1);
    mbar_init(&tfull[1], 1);
    mbar_init(w2bar, 1);
    mbar_init(hbar, 1);
    for (int rd = 0; rd < 3; ++rd) mbar_init(&rbar[rd], 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_trigger();
  if (threadIdx.x == 0) GEMM_TRACE(0);

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------- W1 (weights: never produced by a predecessor)
      tma_prefetch_desc(&tmW1);
      tma_prefetch_desc(&tmW2);
      if (w2_early) load_w2(w2s, &tmW2, w2bar, rank);
      for (int i = 0; i < KB; ++i) {
        const int s = i & 1;
        mbar_wait(&empty[s], ((i >> 1) & 1) ^ 1);
        const uint32_t wdst = smem_addr(r0 + s * kHdStage + kABytes);
        mbar_arrive_expect_tx(&full[s], kHdWBytes);
        tma_load_2d(wdst, &tmW1, &full[s], (kb0 + i) * kBK, 0);
        tma_load_2d(wdst + kHdWBytes / 2, &tmW1, &full[s], (kb0 + i) * kBK, 256);
      }
    }
  } else if (warp == 1) {  // -------------------------------------------- FC1 MMA
    constexpr uint32_t idesc = umma_idesc_bf16_m128(256);
    for (int i = 0; i < KB; ++i) {
      const int s = i & 1;
      mbar_wait(&full[s], (i >> 1) & 1);
      if (i == 0 && lane == 0) GEMM_TRACE(1);
      fence_proxy_async_smem();  // cp.async (generic proxy) rows -> tensor core reads
      tc_fence_after();
      const uint64_t adesc = umma_desc_sw128(smem_addr(r0 + s * kHdStage));
      const uint64_t bdesc = umma_desc_sw128(smem_addr(r0 + s * kHdStage + kABytes));
#pragma unroll
      for (int k = 0; k < kBK / 16; ++k) {
        umma_bf16_elect(tmem_base, adesc + 2 * k, bdesc + 2 * k, idesc, i != 0 || k != 0);
        umma_bf16_elect(tmem_base + 256, adesc + 2 * k, bdesc + (kHdWBytes / 2 >> 4) + 2 * k, idesc,
                        i != 0 || k != 0);
      }
      umma_commit_elect(&empty[s]);
      __syncwarp();
    }
    umma_commit_elect(&tfull[0]);
    __syncwarp();
  } else if (warp == 2) {  // bias slices (weights: no dependency on a predecessor)
    for (int c = lane; c < kHdSlice; c += 32) {
      const int col = (int)rank * kHdSlice + c;
      sb1[c] = p.bias[col];
      sb2[c] = col < p.N ? p.red_bias[col] : 0.0f;
    }
  } else if (warp >= 4) {  // ------------------------------ A gather (one request row per thread)
    pdl_wait();  // features and inv come from the encoders / compaction
    const int r = threadIdx.x - 128;
    const int row = m_tile * kBM + r;
    const int kb_per_mod = p.feat_dim / kBK;
    int cur_k = -1, j = -1;
    for (int i = 0; i < KB; ++i) {
      const int s = i & 1;
      mbar_wait(&empty[s], ((i >> 1) & 1) ^ 1);
      const int kb = kb0 + i;
      const int k = kb / kb_per_mod;
      if (k != cur_k) {
        cur_k = k;
        j = row < p.M ? p.inv[(long long)k * p.inv_ld + row] : -1;
      }
      const __nv_bfloat16* src = j >= 0 ? p.feat[k] + (long long)j * p.feat_dim + (kb - k * kb_per_mod) * kBK : nullptr;
      const uint32_t dst = smem_addr(r0 + s * kHdStage) + r * 128;
#pragma unroll
      for (int c = 0; c < 8; ++c)
        cp_async_16(dst + ((uint32_t)(c ^ (r & 7))) * 16, src ? (const void*)(src + c * 8) : (const void*)p.feat[0],
                    src ? 16u : 0u);
      cp_async_mbar_arrive_noinc(&full[s]);
    }
  }

  // ------------------------------------------------- phase 2: FC1 reduce-scatter
  const int q = warp & 3, half = warp >> 2;
  const int row = 32 * q + lane;
  const uint32_t taddr_row = tmem_base + ((uint32_t)(32 * q) << 16);
  const bool live = 32 * q < valid;  // warp-uniform: its lane quarter holds a request
  mbar_wait(&tfull[0], 0);
  tc_fence_after();
  if (threadIdx.x == 0) GEMM_TRACE(2);
  float acc[32] = {};
  // every CTA's phase-1 use of its window is over once its MMAs completed
  // (tfull), and the barrier inits are visible cluster-wide after this
  cluster_sync_all();
  if (threadIdx.x == 0) GEMM_TRACE(3);
  reduce_scatter(acc, taddr_row, r0, rank, row, half, live, vpad, w2_early ? kHdR0 : kHdWindow, rbar);
  if (threadIdx.x == 0) GEMM_TRACE(4);

  // ------------------------------------------------- phase 3: h chunk + all-gather
  if (threadIdx.x == 0) {  // the window is free cluster-wide (last round's cluster barrier)
    if (!w2_early) load_w2(w2s, &tmW2, w2bar, rank);
    mbar_arrive_expect_tx(hbar, (kHdCL - 1) * vpad * 128);
  }
  uint8_t* hmine = r0 + rank * kHdHChunk;
  if (live) {
    uint32_t hv[16];
#pragma unroll
    for (int c = 0; c < 16; ++c)
      hv[c] = pack_bf16x2(fmaxf(acc[2 * c] + sb1[half * 32 + 2 * c], 0.0f),
                          fmaxf(acc[2 * c + 1] + sb1[half * 32 + 2 * c + 1], 0.0f));
    uint8_t* hrow = hmine + row * 128;
#pragma unroll
    for (int c = 0; c < 4; ++c)
      *reinterpret_cast<uint4*>(hrow + (((uint32_t)(half * 4 + c) ^ (uint32_t)(row & 7)) * 16)) =
          make_uint4(hv[4 * c], hv[4 * c + 1], hv[4 * c + 2], hv[4 * c + 3]);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int j = 1; j < kHdCL; ++j) {  // rows [0, vpad) of the chunk are one contiguous run
      const uint32_t o = (rank + j) % kHdCL;
      bulk_s2s_cluster(mapa_shared(smem_addr(hmine), o), smem_addr(hmine), vpad * 128, mapa_shared(smem_addr(hbar), o));
    }
  }
  if (warp == 1) {  // ------------------------------------------- FC2 MMA (N = 64, K = 512)
    mbar_wait(hbar, 0);
    mbar_wait(w2bar, 0);
    tc_fence_after();
    constexpr uint32_t idesc = umma_idesc_bf16_m128(kHdSlice);
#pragma unroll 1
    for (int kc = 0; kc < 8; ++kc) {
      const uint64_t adesc = umma_desc_sw128(smem_addr(r0 + kc * kHdHChunk));
      const uint64_t bdesc = umma_desc_sw128(smem_addr(w2s + kc * kHdW2Chunk));
#pragma unroll
      for (int k = 0; k < kBK / 16; ++k) umma_bf16_elect(tmem_base, adesc + 2 * k, bdesc + 2 * k, idesc, kc | k);
    }
    umma_commit_elect(&tfull[1]);
    __syncwarp();
  }
  mbar_wait(hbar, 0);
  // every CTA holds all 8 h chunks: no bulk copy reads a peer's shared
  // memory after this barrier, so any CTA may exit once it is done
  cluster_sync_all();
  mbar_wait(&tfull[1], 0);
  tc_fence_after();
  if (threadIdx.x == 0) GEMM_TRACE(5);

  // ------------------------------------------------- phase 4: logits columns [64 r, 64 r + 64)
  if (live) {
    uint32_t v[32];
    tmem_ld_32x32b_x32(taddr_row + half * 32, v);
    tmem_wait_ld();
    const int col0 = (int)rank * kHdSlice + half * 32;
    if (row < valid) {
      float* out = reinterpret_cast<float*>(p.seg[0].ptr) + (long long)(m_tile * kBM + row) * p.seg[0].ldd +
                   p.seg[0].col0;
#pragma unroll
      for (int c = 0; c < 32; ++c)
        if (col0 + c < p.N) out[col0 + c] = __uint_as_float(v[c]) + sb2[half * 32 + c];
    }
  }
  if (threadIdx.x == 0) GEMM_TRACE(7);
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}


// ---------------------------------------------------------------------------
// Small-pass head (MODE_HEAD_GEMV): with few requests the head is a weight
// stream -- W1 (512 x K bf16, 4 MB at K = 4096) dwarfs the features -- and the
// cluster head above reads it with 8 SMs.  Here ONE launch of 128 CTAs
// streams it: FC1 gives each CTA 4 hidden rows (every thread holds its
// 8-element K chunks of those rows in registers, loaded -- with the CTA's FC2
// rows -- before griddepcontrol.wait, so the stream overlaps the previous
// kernel's tail), gathers each request's concatenated features through inv
// (absent modality = zero K block, profile.py:157-159) with all of a group's
// loads in flight, and reduces 4 rows x Q requests per pass with a
// multi-sum butterfly (warp_reduce_multi).  h is rounded to bf16 (the
// unfused path's rounding point).  A grid barrier (all 128 CTAs co-resident)
// replaces a second launch; FC2 then gives each warp one class at a time.
// Every output has one producer in a fixed order: reruns are bitwise
// identical.
constexpr int kGvThreads = 256;
constexpr int kGvRows = 4;      // hidden rows per FC1 CTA
constexpr int kGvMaxCh = 2;     // K <= 2 * 256 * 8 = 4096

__device__ __forceinline__ void bf16x8_to_f32(const uint4& u, float (&f)[8]) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}

// v[j] on entry: this lane's partial of sum j (V sums, V a power of two <=
// 32); on return v[0] = the warp's total of sum (lane & (V - 1)): plain xor
// reductions over the lane bits >= V, then a butterfly transpose-reduce over
// the low bits (V - 1 shuffles instead of V * 5)
template <int V>
__device__ __forceinline__ float warp_reduce_multi(float (&v)[V], int lane) {
#pragma unroll
  for (int off = 16; off >= V; off >>= 1)
#pragma unroll
    for (int j = 0; j < V; ++j) v[j] += __shfl_xor_sync(0xffffffffu, v[j], off);
#pragma unroll
  for (int off = V / 2; off >= 1; off >>= 1) {
    const bool hi = (lane & off) != 0;
#pragma unroll
    for (int j = 0; j < off; ++j) {
      const float keep = hi ? v[j + off] : v[j];
      const float send = hi ? v[j] : v[j + off];
      v[j] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  return v[0];
}

// grid-wide barrier for a grid whose CTAs are all co-resident (128 CTAs of
// one 256-thread block per SM at most): arrive on a counter, the last
// arriver resets it and bumps the generation word the others spin on, so the
// two words are ready for the next launch (graph replays) without a memset
__device__ __forceinline__ void grid_barrier(unsigned* sync) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = sync + 1;
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(sync, 1u) == gridDim.x - 1) {
      atomicExch(sync, 0u);
      __threadfence();
      atomicAdd(sync + 1, 1u);
    } else {
      while (*gen == g) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

// Q: requests per reduction pass (1, 2, 4 or 8, picked from M at launch so a
// one-request head does one request's FMAs)
template <int Q>
__global__ void __launch_bounds__(kGvThreads) head_gemv_kernel(const GemmParams p, const __nv_bfloat16* __restrict__ W1,
                                                               const __nv_bfloat16* __restrict__ W2, unsigned* sync) {
  __shared__ float red[kGvThreads / 32][32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // FC2 rows of this CTA: warp w takes class blockIdx.x + w * gridDim.x
  // (lane covers K = [8 lane, 8 lane + 8) and [256 + 8 lane, ...))
  const int cls = blockIdx.x + warp * gridDim.x;
  const bool live = cls < p.N;
  uint4 v0 = make_uint4(0, 0, 0, 0), v1 = v0;
  float bias2 = 0.f;
  if (live) {
    const uint4* wr = reinterpret_cast<const uint4*>(W2 + (long long)cls * kHdHidden);
    v0 = __ldg(wr + lane);
    v1 = __ldg(wr + 32 + lane);
    bias2 = __ldg(p.red_bias + cls);
  }
  const int K = p.n_mod * p.feat_dim, nch = K / 8, row0 = blockIdx.x * kGvRows;
  uint4 w[kGvMaxCh][kGvRows];
#pragma unroll
  for (int i = 0; i < kGvMaxCh; ++i) {
    const int c = tid + i * kGvThreads;
#pragma unroll
    for (int rr = 0; rr < kGvRows; ++rr)
      w[i][rr] = c < nch ? __ldg(reinterpret_cast<const uint4*>(W1 + (long long)(row0 + rr) * K) + c)
                         : make_uint4(0, 0, 0, 0);
  }
  pdl_wait();  // features / inv come from the encoders and the compaction
  pdl_trigger();
  int mch[kGvMaxCh], dch[kGvMaxCh];
#pragma unroll
  for (int i = 0; i < kGvMaxCh; ++i) {
    const int c = min(tid + i * kGvThreads, nch - 1);
    mch[i] = (c * 8) / p.feat_dim;
    dch[i] = c * 8 - mch[i] * p.feat_dim;
  }
  constexpr int V1 = kGvRows * Q;
  for (int g0 = 0; g0 < p.M; g0 += Q) {
    // every gather of the group in flight at once: inv rows, then feature chunks
    int src[kGvMaxCh][Q];
#pragma unroll
    for (int i = 0; i < kGvMaxCh; ++i)
#pragma unroll
      for (int q = 0; q < Q; ++q)
        src[i][q] = (g0 + q < p.M && tid + i * kGvThreads < nch) ? __ldg(p.inv + (long long)mch[i] * p.inv_ld + g0 + q)
                                                                 : -1;
    uint4 xv[kGvMaxCh][Q];
#pragma unroll
    for (int i = 0; i < kGvMaxCh; ++i)
#pragma unroll
      for (int q = 0; q < Q; ++q)
        xv[i][q] = src[i][q] >= 0 ? __ldg(reinterpret_cast<const uint4*>(p.feat[mch[i]] + (long long)src[i][q] * p.feat_dim +
                                                                         dch[i]))
                                  : make_uint4(0, 0, 0, 0);  // absent modality: a zero K block
    float acc[V1];
#pragma unroll
    for (int j = 0; j < V1; ++j) acc[j] = 0.f;
#pragma unroll
    for (int i = 0; i < kGvMaxCh; ++i) {
      float wf[kGvRows][8];
#pragma unroll
      for (int rr = 0; rr < kGvRows; ++rr) bf16x8_to_f32(w[i][rr], wf[rr]);
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        float x[8];
        bf16x8_to_f32(xv[i][q], x);
#pragma unroll
        for (int rr = 0; rr < kGvRows; ++rr)
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[rr * Q + q] = fmaf(wf[rr][e], x[e], acc[rr * Q + q]);
      }
    }
    const float part = warp_reduce_multi<V1>(acc, lane);
    if (lane < V1) red[warp][lane] = part;
    __syncthreads();
    if (warp == 0 && lane < V1) {
      float s = 0.f;
#pragma unroll
      for (int k = 0; k < kGvThreads / 32; ++k) s += red[k][lane];
      const int rr = lane / Q, r = g0 + lane % Q, row = row0 + rr;
      if (r < p.M) p.hbuf[(long long)r * kHdHidden + row] = __float2bfloat16_rn(fmaxf(s + p.bias[row], 0.f));
    }
    __syncthreads();
  }
  grid_barrier(sync);  // every h row complete (and visible at L2)
  float* out = reinterpret_cast<float*>(p.seg[0].ptr);
  // classes cls, cls + 8 * grid, ... (the first one's row was prefetched)
  for (int c = cls; c < p.N; c += kGvThreads / 32 * gridDim.x) {
    float bias = bias2;
    if (c != cls) {
      const uint4* wr = reinterpret_cast<const uint4*>(W2 + (long long)c * kHdHidden);
      v0 = __ldg(wr + lane);
      v1 = __ldg(wr + 32 + lane);
      bias = __ldg(p.red_bias + c);
    }
    float wa[8], wb[8];
    bf16x8_to_f32(v0, wa);
    bf16x8_to_f32(v1, wb);
    for (int g0 = 0; g0 < p.M; g0 += Q) {
      uint4 hv[Q][2];  // the group's h chunks in flight at once
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int r = g0 + q;
        const uint4* hr = reinterpret_cast<const uint4*>(p.hbuf + (long long)r * kHdHidden);
        hv[q][0] = r < p.M ? __ldcg(hr + lane) : make_uint4(0, 0, 0, 0);  // L2: written by other CTAs
        hv[q][1] = r < p.M ? __ldcg(hr + 32 + lane) : make_uint4(0, 0, 0, 0);
      }
      float acc[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        float ha[8], hb[8];
        bf16x8_to_f32(hv[q][0], ha);
        bf16x8_to_f32(hv[q][1], hb);
        float a = 0.f;
#pragma unroll
        for (int e = 0; e < 8; ++e) a = fmaf(wa[e], ha[e], a);
#pragma unroll
        for (int e = 0; e < 8; ++e) a = fmaf(wb[e], hb[e], a);
        acc[q] = a;
      }
      const float s = warp_reduce_multi<Q>(acc, lane);
      if (lane < Q && g0 + lane < p.M) out[(long long)(g0 + lane) * p.seg[0].ldd + c] = s + bias;
    }
  }
}

}  // namespace

int launch_fused_head(const GemmPlan* P, cudaStream_t stream) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(fused_head_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kHdSmem);
    attr = true;
  }
  launch_k(fused_head_kernel, dim3(P->grid_x), dim3(kHdThreads), kHdSmem, stream, kHdCL, P->tmA, P->tmB, P->p);
  return check_launch("fused_head_kernel");
}


int launch_head_gemv(const GemmPlan* P, cudaStream_t stream) {
  const GemmParams& p = P->p;
  auto* kern = p.M <= 1 ? head_gemv_kernel<1> : p.M <= 2 ? head_gemv_kernel<2> : p.M <= 4 ? head_gemv_kernel<4>
                                                                                    : head_gemv_kernel<8>;
  launch_k(kern, dim3(P->grid_x), dim3(kGvThreads), 0, stream, 1, p, reinterpret_cast<const __nv_bfloat16*>(P->w_ptr),
           p.residual, reinterpret_cast<unsigned*>(p.ws));
  return check_launch("head_gemv_kernel");
}

}  // namespace mosel

using namespace mosel;

extern "C" int ms_gemm_plan_fused_head(void* plan, const void* const* feat, const int32_t* inv, int inv_ld, int n_mod,
                                       int feat_dim, int M, const void* W1, const float* b1, const void* W2,
                                       const float* b2, int n_classes, float* logits, long long ldo) {
  if (plan == nullptr || feat == nullptr || inv == nullptr || W1 == nullptr || W2 == nullptr || b1 == nullptr ||
      b2 == nullptr || logits == nullptr)
    return set_error(MS_ERR_INVALID, "null pointer");
  if (n_mod < 1 || n_mod > 4 || feat_dim % kBK != 0 || M <= 0 || ldo < n_classes)
    return set_error(MS_ERR_INVALID, "fused head needs 1..4 modalities, feat_dim % 64 == 0, M > 0");
  if (n_classes < 1 || n_classes > kHdHidden || (n_mod * feat_dim) % (kBK * kHdCL) != 0)
    return set_error(MS_ERR_INVALID, "fused head needs classes <= 512 and K % 512 == 0");
  GemmPlan* P = reinterpret_cast<GemmPlan*>(plan);
  memset(P, 0, sizeof(GemmPlan));
  GemmParams& p = P->p;
  p.mode = MODE_FUSED_HEAD;
  p.M = M;
  p.N = n_classes;
  p.bias = b1;
  p.red_bias = b2;
  p.inv = inv;
  p.inv_ld = inv_ld;
  p.n_mod = n_mod;
  p.feat_dim = feat_dim;
  for (int k = 0; k < n_mod; ++k) p.feat[k] = reinterpret_cast<const __nv_bfloat16*>(feat[k]);
  for (int k = n_mod; k < 4; ++k) p.feat[k] = p.feat[0];
  p.nseg = 1;
  p.seg[0] = Seg{0, n_classes, logits, ldo, 0, 0};
  p.out_fp32 = 1;
  const int K = n_mod * feat_dim;
  p.num_kb = K / kBK / kHdCL;
  p.m_tiles = (M + kBM - 1) / kBM;
  cuuint64_t d1[2] = {(cuuint64_t)K, (cuuint64_t)kHdHidden};
  cuuint64_t s1[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {(cuuint32_t)kBK, 256};
  cuuint32_t es[2] = {1, 1};
  int rc = encode_bf16_map(&P->tmB, 2, W1, d1, s1, box, es, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  cuuint64_t d2[2] = {(cuuint64_t)kHdHidden, (cuuint64_t)n_classes};  // rows >= classes: zero fill
  cuuint64_t s2[1] = {(cuuint64_t)kHdHidden * 2};
  cuuint32_t box2[2] = {(cuuint32_t)kBK, (cuuint32_t)kHdSlice};
  rc = encode_bf16_map(&P->tmA, 2, W2, d2, s2, box2, es, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  P->grid_x = p.m_tiles * kHdCL;
  P->grid_y = 1;
  P->smem_bytes = kHdSmem;
  P->tmem_cols = 512;
  return MS_OK;
}

extern "C" int ms_gemm_plan_head_gemv(void* plan, const void* const* feat, const int32_t* inv, int inv_ld, int n_mod,
                                      int feat_dim, int M, const void* W1, const float* b1, const void* W2,
                                      const float* b2, int n_classes, float* logits, long long ldo, void* h,
                                      void* sync) {
  if (plan == nullptr || feat == nullptr || inv == nullptr || W1 == nullptr || W2 == nullptr || b1 == nullptr ||
      b2 == nullptr || logits == nullptr || h == nullptr || sync == nullptr)
    return set_error(MS_ERR_INVALID, "null pointer");
  if (n_mod < 1 || n_mod > 4 || feat_dim % 8 != 0 || M <= 0 || ldo < n_classes || n_classes < 1)
    return set_error(MS_ERR_INVALID, "gemv head needs 1..4 modalities, feat_dim % 8 == 0, M > 0, classes >= 1");
  if (n_mod * feat_dim > kGvMaxCh * kGvThreads * 8) return set_error(MS_ERR_INVALID, "gemv head needs K <= 4096");
  GemmPlan* P = reinterpret_cast<GemmPlan*>(plan);
  memset(P, 0, sizeof(GemmPlan));
  GemmParams& p = P->p;
  p.mode = MODE_HEAD_GEMV;
  p.M = M;
  p.N = n_classes;
  p.bias = b1;
  p.red_bias = b2;
  p.inv = inv;
  p.inv_ld = inv_ld;
  p.n_mod = n_mod;
  p.feat_dim = feat_dim;
  for (int k = 0; k < n_mod; ++k) p.feat[k] = reinterpret_cast<const __nv_bfloat16*>(feat[k]);
  for (int k = n_mod; k < 4; ++k) p.feat[k] = p.feat[0];
  p.nseg = 1;
  p.seg[0] = Seg{0, n_classes, logits, ldo, 0, 0};
  p.out_fp32 = 1;
  p.hbuf = reinterpret_cast<__nv_bfloat16*>(h);
  p.ws = reinterpret_cast<float*>(sync);  // two zeroed 32-bit words: barrier count, generation
  p.residual = reinterpret_cast<const __nv_bfloat16*>(W2);  // [classes, 512] rows
  P->w_ptr = W1;                                            // [512, K] rows
  P->grid_x = kHdHidden / kGvRows;
  P->grid_y = 1;
  return MS_OK;
}
