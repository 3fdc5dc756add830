// Transformer-tower pieces for configs[2] (ViT-B/16 image tower + BERT-base
// text tower).  The dense layers (QKV, out-proj + residual,
// MLP with GELU, pooler with tanh) are tcgen05 GEMM plans (gemm.cu); this file
// holds the rest:
//   * layernorm_kernel      — one warp per row, fp32 statistics, bf16 out,
//                             arbitrary input/output row strides (so the
//                             final LN can read only the CLS rows)
//   * attention_tc_kernel   — fused softmax(Q K^T * scale) V per (sequence,
//                             head): both contractions tcgen05.mma with S and
//                             the output in TMEM, P staged as the SMEM A
//                             operand (L <= 256 keys)
//   * patchify_kernel       — NHWC image -> [patches, (kh, kw, c)] rows
//   * vit_embed_kernel      — [CLS | patch embeddings] + position embeddings
//   * bert_embed_kernel     — word + position + type embeddings, then LN
#include <cstdint>

#include "mosel_b200.h"
#include "ptx.cuh"
#include "runtime.h"

namespace mosel {

// ------------------------------------------------------------- LayerNorm
// C % 256 == 0: each lane owns C/256 chunks of 8 contiguous channels.
template <int CH>
__device__ __forceinline__ void ln_row(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ y,
                                       const float* __restrict__ gamma, const float* __restrict__ beta, int C,
                                       float eps, int lane) {
  float v[CH][8];
  float sum = 0.0f;
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const uint4 q = *reinterpret_cast<const uint4*>(x + (c * 32 + lane) * 8);
    const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&q);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      v[c][j] = __bfloat162float(e[j]);
      sum += v[c][j];
    }
  }
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const float mean = sum / (float)C;
  float var = 0.0f;
#pragma unroll
  for (int c = 0; c < CH; ++c)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float d = v[c][j] - mean;
      var += d * d;
    }
  for (int o = 16; o > 0; o >>= 1) var += __shfl_xor_sync(0xffffffffu, var, o);
  const float rstd = rsqrtf(var / (float)C + eps);
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const int base = (c * 32 + lane) * 8;
    uint32_t pk[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float a = (v[c][2 * j] - mean) * rstd * gamma[base + 2 * j] + beta[base + 2 * j];
      const float b = (v[c][2 * j + 1] - mean) * rstd * gamma[base + 2 * j + 1] + beta[base + 2 * j + 1];
      pk[j] = pack_bf16x2(a, b);
    }
    *reinterpret_cast<uint4*>(y + base) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
  }
}

template <int CH>
__global__ void layernorm_kernel(const __nv_bfloat16* __restrict__ X, long long ldx, long long rows,
                                 const float* __restrict__ gamma, const float* __restrict__ beta,
                                 __nv_bfloat16* __restrict__ Y, long long ldy, int C, float eps) {
  pdl_trigger();
  pdl_wait();
  const long long row = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  if (row >= rows) return;
  ln_row<CH>(X + row * ldx, Y + row * ldy, gamma, beta, C, eps, threadIdx.x & 31);
}

// ------------------------------------------------------------- attention
// softmax(Q K^T * scale) V on the 5th-gen tensor cores, one CTA per
// (head, sequence, 128-query block), L <= 256 keys (ViT-B/16: 197, BERT: 40):
//   TMA    Q block [128 x 64], K [Lk16 x 64] (SW128 K-major) and V rows
//          (unswizzled staging) from the packed QKV activations;
//   V^T    all 128 threads transpose V into K-major SW128 chunks of 64 keys
//          (the B operand of P V), zero past L;
//   S      tcgen05.mma M=128, N=Lk16, K=64 -> TMEM (one query row per lane);
//   P      each thread reads its row from TMEM (tcgen05.ld), masks keys >= L,
//          exp2 with the running max, sums in fp32 and stores P (bf16) into
//          SW128 K-major SMEM chunks -- the A operand of the second MMA;
//   O      tcgen05.mma M=128, N=64, K=Lk64 into TMEM columns the consumed S
//          occupied; epilogue scales by 1/rowsum and stores bf16 rows.
// Both contractions are UMMA (UTCHMMA).  One CTA per (head, sequence, query
// block of 128); Q, K and the V staging rows share the P region, so a CTA
// takes <= 100 KB and two run per SM; S rows come out of TMEM 64 columns per
// round trip.
constexpr int kHd = 64;    // head dim
constexpr int kAttnMaxL = 256;
constexpr int kAttnThreads = 256;  // 8 warps: 2 per TMEM lane quarter, each half of the key columns

__device__ __forceinline__ float fast_exp2(float x) {  // MUFU.EX2 (ftz): p in (0, 1]
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

struct AttnMaps {
  CUtensorMap q, k, v;
};

__global__ void __launch_bounds__(kAttnThreads, 1)
    attention_tc_kernel(const __grid_constant__ AttnMaps maps, int L, int Lk16, int Lk64, int D,
                        __nv_bfloat16* __restrict__ out, long long ldo, float scale_log2) {
  // smem: [V^T chunks | P chunks]; Q, K and the V staging rows live inside the
  // P region (dead before P is written), so a CTA needs <= 100 KB: two per SM
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
  const int nchunk = Lk64 / 64;
  const int kbytes = (Lk16 * 128 + 1023) & ~1023;
  uint8_t* sVT = smem;                                  // nchunk x (64 x 128 B)
  uint8_t* sP = sVT + nchunk * 8192;                    // P: nchunk x (128 x 128 B)
  uint8_t* sQ = sP;                                     // 16 KB   (inside P)
  uint8_t* sK = sQ + 128 * 128;                         // Lk16 x 128 B
  uint8_t* sVs = sK + kbytes;                           // V staging rows, Lk16 x 128 B
  const int pbytes = max(nchunk * 16384, 128 * 128 + 2 * kbytes);
  uint64_t* bar_ld = reinterpret_cast<uint64_t*>(sP + pbytes);
  uint64_t* bar_mma = bar_ld + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_mma + 1);
  __shared__ float s_red[2][128];  // per-half row max, then row sum
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int h = blockIdx.x;
  const long long row0 = (long long)blockIdx.y * L;
  const int q0 = blockIdx.z * 128;  // this CTA's query block

  if (warp == 0) tmem_alloc(tmem_slot, 256);
  if (tid == 0) {
    mbar_init(bar_ld, 1);
    mbar_init(bar_mma, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();
  if (tid == 0) {
    mbar_arrive_expect_tx(bar_ld, 2u * (uint32_t)Lk16 * 128u + 128u * 128u);
    tma_load_2d(smem_addr(sQ), &maps.q, bar_ld, h * kHd, (int)(row0 + q0));
    tma_load_2d(smem_addr(sK), &maps.k, bar_ld, D + h * kHd, (int)row0);
    tma_load_2d(smem_addr(sVs), &maps.v, bar_ld, 2 * D + h * kHd, (int)row0);
  }
  mbar_wait(bar_ld, 0);
  tc_fence_after();
  const uint32_t idesc_s = umma_idesc_bf16_m128((uint32_t)Lk16);
  const uint32_t idesc_o = umma_idesc_bf16_m128((uint32_t)kHd);
  if (warp == 0) {  // S = Q K^T (4 K=16 steps over the head dim), overlaps the V transpose
    const uint64_t qd = umma_desc_sw128(smem_addr(sQ)), kd = umma_desc_sw128(smem_addr(sK));
#pragma unroll
    for (int k = 0; k < kHd / 16; ++k) umma_bf16_elect(tmem, qd + 2 * k, kd + 2 * k, idesc_s, k != 0);
    umma_commit_elect(bar_mma);
  }
  // V^T: element (d, key) of chunk key/64 at d*128 + swizzled 16-B group of key%64
  const __nv_bfloat16* sV = reinterpret_cast<const __nv_bfloat16*>(sVs);
  for (int idx = tid; idx < kHd * (Lk64 / 8); idx += kAttnThreads) {
    const int d = idx & (kHd - 1), key0 = (idx >> 6) * 8;
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int k0 = key0 + 2 * j;
      const __nv_bfloat16 lo = k0 < L ? sV[k0 * kHd + d] : __float2bfloat16(0.0f);
      const __nv_bfloat16 hi = k0 + 1 < L ? sV[(k0 + 1) * kHd + d] : __float2bfloat16(0.0f);
      w[j] = (uint32_t)__bfloat16_as_ushort(lo) | ((uint32_t)__bfloat16_as_ushort(hi) << 16);
    }
    const int grp = (key0 & 63) >> 3;
    *reinterpret_cast<uint4*>(sVT + (key0 >> 6) * 8192 + d * 128 + ((grp ^ (d & 7)) << 4)) =
        make_uint4(w[0], w[1], w[2], w[3]);
  }
  mbar_wait(bar_mma, 0);
  tc_fence_after();
  __syncthreads();  // V staging, Q and K consumed: the P region is free

  // warp w: TMEM lane quarter w % 4 (its 32 query rows), key-column half w / 4
  const int quarter = warp & 3, half = warp >> 2;
  const int r = quarter * 32 + lane;  // this thread's query row in the block (TMEM lane)
  const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16);
  uint8_t* prow = sP + r * 128;
  const int ch = Lk64 / 2;  // columns per half (a multiple of 32)
  const int cbeg = half * ch, cend = cbeg + ch;
  // row max over the valid keys: up to 64 columns per TMEM round trip
  float mx = -INFINITY;
  for (int c0 = cbeg; c0 < cend; c0 += 64) {
    uint32_t v[4][16];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (c0 + 16 * u < min(cend, Lk16)) tmem_ld_32x32b_x16(taddr + (uint32_t)(c0 + 16 * u), v[u]);
    tmem_wait_ld();
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (c0 + 16 * u + j < min(cend, L)) mx = fmaxf(mx, __uint_as_float(v[u][j]));
  }
  s_red[half][r] = mx;
  __syncthreads();
  mx = fmaxf(s_red[0][r], s_red[1][r]);
  const float mxs = mx * scale_log2;
  float sum = 0.0f;
  for (int c0 = cbeg; c0 < cend; c0 += 64) {
    uint32_t v[4][16];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (c0 + 16 * u < min(cend, Lk16)) tmem_ld_32x32b_x16(taddr + (uint32_t)(c0 + 16 * u), v[u]);
    tmem_wait_ld();
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (c0 + 16 * u >= cend) break;
      uint8_t* chunk = prow + ((c0 + 16 * u) >> 6) * 16384;  // a half may start mid-chunk (Lk64 = 192)
      uint32_t pk[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int c = c0 + 16 * u + 2 * j;
        const float p0 = c < L ? fast_exp2(__uint_as_float(v[u][2 * j]) * scale_log2 - mxs) : 0.0f;
        const float p1 = c + 1 < L ? fast_exp2(__uint_as_float(v[u][2 * j + 1]) * scale_log2 - mxs) : 0.0f;
        sum += p0 + p1;
        pk[j] = pack_bf16x2(p0, p1);
      }
      const int g0 = ((c0 + 16 * u) & 63) >> 3;
      *reinterpret_cast<uint4*>(chunk + ((g0 ^ (r & 7)) << 4)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
      *reinterpret_cast<uint4*>(chunk + (((g0 + 1) ^ (r & 7)) << 4)) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
    }
  }
  __syncthreads();  // every half has read its max from s_red
  s_red[half][r] = sum;
  tc_fence_before();
  fence_proxy_async_smem();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {  // O = P V over the key chunks, into the consumed S columns
    for (int kc = 0; kc < nchunk; ++kc) {
      const uint64_t pd = umma_desc_sw128(smem_addr(sP + kc * 16384));
      const uint64_t vd = umma_desc_sw128(smem_addr(sVT + kc * 8192));
#pragma unroll
      for (int k = 0; k < 4; ++k) umma_bf16_elect(tmem, pd + 2 * k, vd + 2 * k, idesc_o, (kc | k) != 0);
    }
    umma_commit_elect(bar_mma);
  }
  mbar_wait(bar_mma, 1);
  tc_fence_after();
  sum = s_red[0][r] + s_red[1][r];
  const float inv = sum > 0.0f ? 1.0f / sum : 0.0f;
  const int q = q0 + r;
  uint32_t v[32];
  tmem_ld_32x32b_x32(taddr + (uint32_t)(half * 32), v);  // this half's 32 output dims
  tmem_wait_ld();
  if (q < L) {
    uint4* dst = reinterpret_cast<uint4*>(out + (row0 + q) * ldo + h * kHd + half * 32);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t* w = &v[8 * j];
      dst[j] = make_uint4(pack_bf16x2(__uint_as_float(w[0]) * inv, __uint_as_float(w[1]) * inv),
                          pack_bf16x2(__uint_as_float(w[2]) * inv, __uint_as_float(w[3]) * inv),
                          pack_bf16x2(__uint_as_float(w[4]) * inv, __uint_as_float(w[5]) * inv),
                          pack_bf16x2(__uint_as_float(w[6]) * inv, __uint_as_float(w[7]) * inv));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

// ------------------------------------------------------------- embeddings
// NHWC image [n, S, S, C] -> rows [n * (S/P)^2, P*P*C], K order (kh, kw, c);
// requires P*C % 8 == 0 (16-B vectors along each patch row).
__global__ void patchify_kernel(const __nv_bfloat16* __restrict__ X, int n, int S, int C, int P,
                                __nv_bfloat16* __restrict__ Y) {
  pdl_trigger();
  pdl_wait();
  const int G = S / P, row_elems = P * P * C, c8 = row_elems / 8;
  const long long total = (long long)n * G * G * c8;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int chunk = (int)(t % c8);
    const long long patch = t / c8;
    const int pw = (int)(patch % G), ph = (int)((patch / G) % G);
    const long long img = patch / (G * G);
    const int e = chunk * 8, kh = e / (P * C), rem = e - kh * P * C;
    const __nv_bfloat16* src = X + ((img * S + ph * P + kh) * S + pw * P) * C + rem;
    reinterpret_cast<uint4*>(Y)[t] = *reinterpret_cast<const uint4*>(src);
  }
}

// tokens[s*L + 0] = cls + pos[0]; tokens[s*L + 1 + p] = pe[s*(L-1) + p] + pos[1 + p]
__global__ void vit_embed_kernel(const __nv_bfloat16* __restrict__ pe, const __nv_bfloat16* __restrict__ cls,
                                 const __nv_bfloat16* __restrict__ pos, int n, int L, int D,
                                 __nv_bfloat16* __restrict__ tok) {
  pdl_trigger();
  pdl_wait();
  const int d8 = D / 8;
  const long long total = (long long)n * L * d8;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(t % d8) * 8;
    const long long r = t / d8;
    const int i = (int)(r % L);
    const long long s = r / L;
    const uint4 a = i == 0 ? *reinterpret_cast<const uint4*>(cls + c)
                           : *reinterpret_cast<const uint4*>(pe + (s * (L - 1) + i - 1) * D + c);
    const uint4 b = *reinterpret_cast<const uint4*>(pos + (long long)i * D + c);
    const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
    const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&b);
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
      o[j] = pack_bf16x2(__bfloat162float(a2[j].x) + __bfloat162float(b2[j].x),
                         __bfloat162float(a2[j].y) + __bfloat162float(b2[j].y));
    reinterpret_cast<uint4*>(tok)[t] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// one warp per token: x = word[id] + pos[t] + type[0] (fp32), then LayerNorm
template <int CH>
__global__ void bert_embed_kernel(const int32_t* __restrict__ ids, long long n_tok, int L,
                                  const __nv_bfloat16* __restrict__ word, const __nv_bfloat16* __restrict__ pos,
                                  const __nv_bfloat16* __restrict__ type0, const float* __restrict__ gamma,
                                  const float* __restrict__ beta, __nv_bfloat16* __restrict__ Y, int D, float eps) {
  pdl_trigger();
  pdl_wait();
  const long long tok = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  if (tok >= n_tok) return;
  const int lane = threadIdx.x & 31;
  const int t = (int)(tok % L);
  const __nv_bfloat16* w = word + (long long)ids[tok] * D;
  const __nv_bfloat16* p = pos + (long long)t * D;
  float v[CH][8];
  float sum = 0.0f;
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const int off = (c * 32 + lane) * 8;
    const uint4 a = *reinterpret_cast<const uint4*>(w + off);
    const uint4 b = *reinterpret_cast<const uint4*>(p + off);
    const uint4 e = *reinterpret_cast<const uint4*>(type0 + off);
    const __nv_bfloat16* ae = reinterpret_cast<const __nv_bfloat16*>(&a);
    const __nv_bfloat16* be = reinterpret_cast<const __nv_bfloat16*>(&b);
    const __nv_bfloat16* ee = reinterpret_cast<const __nv_bfloat16*>(&e);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      v[c][j] = __bfloat162float(ae[j]) + __bfloat162float(be[j]) + __bfloat162float(ee[j]);
      sum += v[c][j];
    }
  }
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const float mean = sum / (float)D;
  float var = 0.0f;
#pragma unroll
  for (int c = 0; c < CH; ++c)
#pragma unroll
    for (int j = 0; j < 8; ++j) var += (v[c][j] - mean) * (v[c][j] - mean);
  for (int o = 16; o > 0; o >>= 1) var += __shfl_xor_sync(0xffffffffu, var, o);
  const float rstd = rsqrtf(var / (float)D + eps);
  __nv_bfloat16* y = Y + tok * D;
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const int off = (c * 32 + lane) * 8;
    uint32_t pk[4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
      pk[j] = pack_bf16x2((v[c][2 * j] - mean) * rstd * gamma[off + 2 * j] + beta[off + 2 * j],
                          (v[c][2 * j + 1] - mean) * rstd * gamma[off + 2 * j + 1] + beta[off + 2 * j + 1]);
    *reinterpret_cast<uint4*>(y + off) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
  }
}

static int grid_cap(long long work, int threads) {
  long long b = (work + threads - 1) / threads;
  if (b > 148LL * 32) b = 148LL * 32;
  return b < 1 ? 1 : (int)b;
}

int run_layernorm(const void* X, long long ldx, long long rows, const float* gamma, const float* beta, void* Y,
                  long long ldy, int C, float eps, cudaStream_t st) {
  if (C % 256 != 0 || C > 2048 || ldx % 8 != 0 || ldy % 8 != 0)
    return set_error(MS_ERR_INVALID, "layernorm: C % 256 == 0, C <= 2048, strides % 8 == 0");
  if (rows <= 0) return MS_OK;
  const long long blocks = (rows * 32 + 255) / 256;
  auto Xp = reinterpret_cast<const __nv_bfloat16*>(X);
  auto Yp = reinterpret_cast<__nv_bfloat16*>(Y);
  switch (C / 256) {
    case 1: launch_k(layernorm_kernel<1>, dim3((unsigned)blocks), dim3(256), 0, st, 1, Xp, ldx, rows, gamma, beta, Yp, ldy, C, eps); break;
    case 2: launch_k(layernorm_kernel<2>, dim3((unsigned)blocks), dim3(256), 0, st, 1, Xp, ldx, rows, gamma, beta, Yp, ldy, C, eps); break;
    case 3: launch_k(layernorm_kernel<3>, dim3((unsigned)blocks), dim3(256), 0, st, 1, Xp, ldx, rows, gamma, beta, Yp, ldy, C, eps); break;
    case 4: launch_k(layernorm_kernel<4>, dim3((unsigned)blocks), dim3(256), 0, st, 1, Xp, ldx, rows, gamma, beta, Yp, ldy, C, eps); break;
    default: return set_error(MS_ERR_INVALID, "layernorm: unsupported C");
  }
  return check_launch("layernorm_kernel");
}

int run_attention(const void* qkv, long long ld, int L, int H, int n_seq, void* out, long long ldo, float scale,
                  cudaStream_t st) {
  if (ld % 8 != 0 || ldo % 8 != 0 || L < 1 || H < 1 || n_seq < 0)
    return set_error(MS_ERR_INVALID, "attention: bad shape/stride");
  if (L > kAttnMaxL) return set_error(MS_ERR_INVALID, "attention: sequence length above 256 keys");
  if (n_seq == 0) return MS_OK;
  const int D = H * kHd, Lk16 = (L + 15) / 16 * 16, Lk64 = (L + 63) / 64 * 64;
  AttnMaps maps;
  const cuuint64_t dims[2] = {(cuuint64_t)(3 * D), (cuuint64_t)n_seq * L};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  const cuuint32_t es[2] = {1, 1};
  const cuuint32_t bq[2] = {kHd, 128}, bk[2] = {kHd, (cuuint32_t)Lk16};
  int rc = encode_bf16_map(&maps.q, 2, qkv, dims, strides, bq, es, CU_TENSOR_MAP_SWIZZLE_128B);
  if (!rc) rc = encode_bf16_map(&maps.k, 2, qkv, dims, strides, bk, es, CU_TENSOR_MAP_SWIZZLE_128B);
  if (!rc) rc = encode_bf16_map(&maps.v, 2, qkv, dims, strides, bk, es, CU_TENSOR_MAP_SWIZZLE_NONE);
  if (rc) return rc;
  const int kbytes = (Lk16 * 128 + 1023) & ~1023;
  const int pbytes = (Lk64 / 64) * 16384 > 128 * 128 + 2 * kbytes ? (Lk64 / 64) * 16384 : 128 * 128 + 2 * kbytes;
  const int smem = 1024 + (Lk64 / 64) * 8192 + pbytes + 64;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attention_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  launch_k(attention_tc_kernel, dim3(H, n_seq, (L + 127) / 128), dim3(kAttnThreads), smem, st, 1, maps, L, Lk16,
           Lk64, D,
           reinterpret_cast<__nv_bfloat16*>(out), ldo, scale * 1.4426950408889634f);
  return check_launch("attention_tc_kernel");
}

int run_patchify(const void* X, int n, int S, int C, int P, void* Y, cudaStream_t st) {
  if ((P * C) % 8 != 0 || S % P != 0) return set_error(MS_ERR_INVALID, "patchify: P*C % 8 == 0, S % P == 0");
  const long long work = (long long)n * (S / P) * (S / P) * P * P * C / 8;
  launch_k(patchify_kernel, dim3(grid_cap(work, 256)), dim3(256), 0, st, 1, reinterpret_cast<const __nv_bfloat16*>(X), n, S, C, P,
                                                       reinterpret_cast<__nv_bfloat16*>(Y));
  return check_launch("patchify_kernel");
}

int run_vit_embed(const void* pe, const void* cls, const void* pos, int n, int L, int D, void* tok, cudaStream_t st) {
  if (D % 8 != 0) return set_error(MS_ERR_INVALID, "vit_embed: D % 8 == 0");
  const long long work = (long long)n * L * D / 8;
  launch_k(vit_embed_kernel, dim3(grid_cap(work, 256)), dim3(256), 0, st, 1, 
      reinterpret_cast<const __nv_bfloat16*>(pe), reinterpret_cast<const __nv_bfloat16*>(cls),
      reinterpret_cast<const __nv_bfloat16*>(pos), n, L, D, reinterpret_cast<__nv_bfloat16*>(tok));
  return check_launch("vit_embed_kernel");
}

int run_bert_embed(const int32_t* ids, long long n_tok, int L, const void* word, const void* pos, const void* type0,
                   const float* gamma, const float* beta, void* Y, int D, float eps, cudaStream_t st) {
  if (D != 768) return set_error(MS_ERR_INVALID, "bert_embed: D must be 768");
  if (n_tok <= 0) return MS_OK;
  const long long blocks = (n_tok * 32 + 255) / 256;
  launch_k(bert_embed_kernel<3>, dim3((unsigned)blocks), dim3(256), 0, st, 1, ids, n_tok, L, reinterpret_cast<const __nv_bfloat16*>(word),
                                               reinterpret_cast<const __nv_bfloat16*>(pos),
                                               reinterpret_cast<const __nv_bfloat16*>(type0), gamma, beta,
                                               reinterpret_cast<__nv_bfloat16*>(Y), D, eps);
  return check_launch("bert_embed_kernel");
}

}  // namespace mosel

using namespace mosel;

extern "C" {

int ms_layernorm(const void* X, long long ldx, long long rows, const float* gamma, const float* beta, void* Y,
                 long long ldy, int C, float eps, void* stream) {
  return run_layernorm(X, ldx, rows, gamma, beta, Y, ldy, C, eps, reinterpret_cast<cudaStream_t>(stream));
}

int ms_attention(const void* qkv, long long ld, int L, int H, int n_seq, void* out, long long ldo, float scale,
                 void* stream) {
  return run_attention(qkv, ld, L, H, n_seq, out, ldo, scale, reinterpret_cast<cudaStream_t>(stream));
}

int ms_patchify(const void* X, int n, int S, int C, int P, void* Y, void* stream) {
  return run_patchify(X, n, S, C, P, Y, reinterpret_cast<cudaStream_t>(stream));
}

int ms_vit_embed(const void* pe, const void* cls, const void* pos, int n, int L, int D, void* tok, void* stream) {
  return run_vit_embed(pe, cls, pos, n, L, D, tok, reinterpret_cast<cudaStream_t>(stream));
}

int ms_bert_embed(const int32_t* ids, long long n_tok, int L, const void* word, const void* pos, const void* type0,
                  const float* gamma, const float* beta, void* Y, int D, float eps, void* stream) {
  return run_bert_embed(ids, n_tok, L, word, pos, type0, gamma, beta, Y, D, eps,
                        reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
