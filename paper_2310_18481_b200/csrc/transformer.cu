// Transformer-tower pieces for configs[2] (ViT-B/16 image tower + BERT-base
// text tower).  The dense layers (QKV, out-proj + residual,
// MLP with GELU, pooler with tanh) are tcgen05 GEMM plans (gemm.cu); this file
// holds the rest:
//   * layernorm_kernel      — one warp per row, fp32 statistics, bf16 out,
//                             arbitrary input/output row strides (so the
//                             final LN can read only the CLS rows)
//   * attention_kernel      — fused softmax(Q K^T * scale) V per (sequence,
//                             head, 64-query block), FlashAttention-2 style
//                             online softmax on mma.sync m16n8k16 bf16 tensor
//                             ops with ldmatrix fragments; attention is ~4 %
//                             of ViT-B FLOPs, the rest is on tcgen05
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
constexpr int kHd = 64;    // head dim
constexpr int kBq = 64;    // queries per block (4 warps x 16)
constexpr int kBk = 64;    // keys per iteration
constexpr int kPad = 8;    // smem row padding (bank-conflict-free ldmatrix)

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma_bf16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// qkv rows: [Q(H*64) | K(H*64) | V(H*64)] per token, row stride ld;
// out rows: H*64 per token, row stride ldo.  grid (ceil(L/64), H, n_seq).
__global__ void __launch_bounds__(128) attention_kernel(const __nv_bfloat16* __restrict__ qkv, long long ld, int L,
                                                        int H, __nv_bfloat16* __restrict__ out, long long ldo,
                                                        float scale_log2) {
  pdl_trigger();
  pdl_wait();
  __shared__ __align__(16) __nv_bfloat16 sQ[kBq][kHd + kPad];
  __shared__ __align__(16) __nv_bfloat16 sK[kBk][kHd + kPad];
  __shared__ __align__(16) __nv_bfloat16 sV[kBk][kHd + kPad];
  const int qb = blockIdx.x, h = blockIdx.y;
  const long long seq = blockIdx.z;
  const __nv_bfloat16* base = qkv + seq * L * ld;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int D = H * kHd;

  for (int i = tid; i < kBq * kHd / 8; i += 128) {
    const int r = i >> 3, c8 = (i & 7) * 8;
    const int q = qb * kBq + r;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (q < L) v = *reinterpret_cast<const uint4*>(base + (long long)q * ld + h * kHd + c8);
    *reinterpret_cast<uint4*>(&sQ[r][c8]) = v;
  }
  __syncthreads();
  // Q fragments for this warp's 16 rows, 4 k-steps of 16 dims
  uint32_t qf[4][4];
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    const int r = warp * 16 + (lane & 15), c = ks * 16 + (lane >> 4) * 8;
    ldsm_x4(smem_addr(&sQ[r][c]), qf[ks][0], qf[ks][1], qf[ks][2], qf[ks][3]);
  }
  float o[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.0f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.0f, l1 = 0.0f;
  const int g = lane >> 2, t4 = lane & 3;

  for (int k0 = 0; k0 < L; k0 += kBk) {
    __syncthreads();
    for (int i = tid; i < kBk * kHd / 8; i += 128) {
      const int r = i >> 3, c8 = (i & 7) * 8;
      const int k = k0 + r;
      uint4 kv = make_uint4(0, 0, 0, 0), vv = make_uint4(0, 0, 0, 0);
      if (k < L) {
        kv = *reinterpret_cast<const uint4*>(base + (long long)k * ld + D + h * kHd + c8);
        vv = *reinterpret_cast<const uint4*>(base + (long long)k * ld + 2 * D + h * kHd + c8);
      }
      *reinterpret_cast<uint4*>(&sK[r][c8]) = kv;
      *reinterpret_cast<uint4*>(&sV[r][c8]) = vv;
    }
    __syncthreads();
    // S = Q K^T : 16 rows x 64 keys (8 n-tiles of 8 keys)
    float sc[8][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.0f;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
#pragma unroll
      for (int np = 0; np < 4; ++np) {  // two n-tiles per ldmatrix.x4
        uint32_t b0, b1, b2, b3;
        const int r = np * 16 + (lane & 7) + ((lane >> 4) << 3), c = ks * 16 + ((lane >> 3) & 1) * 8;
        ldsm_x4(smem_addr(&sK[r][c]), b0, b1, b2, b3);
        mma_bf16(sc[2 * np], qf[ks], b0, b1);
        mma_bf16(sc[2 * np + 1], qf[ks], b2, b3);
      }
    }
    // mask keys beyond L, online softmax (rows g and g+8 of the warp tile)
    float mx0 = m0, mx1 = m1;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const int kc = k0 + nt * 8 + 2 * t4;
      if (kc >= L) sc[nt][0] = sc[nt][2] = -INFINITY;
      if (kc + 1 >= L) sc[nt][1] = sc[nt][3] = -INFINITY;
      mx0 = fmaxf(mx0, fmaxf(sc[nt][0], sc[nt][1]) * scale_log2);
      mx1 = fmaxf(mx1, fmaxf(sc[nt][2], sc[nt][3]) * scale_log2);
    }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
    const float a0 = exp2f(m0 - mx0), a1 = exp2f(m1 - mx1);
    m0 = mx0;
    m1 = mx1;
    float s0 = 0.0f, s1 = 0.0f;
    uint32_t pf[8][2];  // P as bf16 pairs: [n-tile][row g / row g+8]
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const float p00 = exp2f(sc[nt][0] * scale_log2 - m0), p01 = exp2f(sc[nt][1] * scale_log2 - m0);
      const float p10 = exp2f(sc[nt][2] * scale_log2 - m1), p11 = exp2f(sc[nt][3] * scale_log2 - m1);
      s0 += p00 + p01;
      s1 += p10 + p11;
      pf[nt][0] = pack_bf16x2(p00, p01);
      pf[nt][1] = pack_bf16x2(p10, p11);
    }
    l0 = l0 * a0 + s0;
    l1 = l1 * a1 + s1;
#pragma unroll
    for (int dt = 0; dt < 8; ++dt) {
      o[dt][0] *= a0;
      o[dt][1] *= a0;
      o[dt][2] *= a1;
      o[dt][3] *= a1;
    }
    // O += P V : k = keys (4 steps of 16), n = 64 dims (8 tiles)
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const uint32_t af[4] = {pf[2 * kk][0], pf[2 * kk][1], pf[2 * kk + 1][0], pf[2 * kk + 1][1]};
#pragma unroll
      for (int dp = 0; dp < 4; ++dp) {  // two dim tiles per ldmatrix.x4.trans
        uint32_t b0, b1, b2, b3;
        const int r = kk * 16 + (lane & 15), c = dp * 16 + (lane >> 4) * 8;
        ldsm_x4_t(smem_addr(&sV[r][c]), b0, b1, b2, b3);
        mma_bf16(o[2 * dp], af, b0, b1);
        mma_bf16(o[2 * dp + 1], af, b2, b3);
      }
    }
  }
  // finalize: row sums across the quad, normalise, store
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const float inv0 = l0 > 0.0f ? 1.0f / l0 : 0.0f, inv1 = l1 > 0.0f ? 1.0f / l1 : 0.0f;
  const int q0 = qb * kBq + warp * 16 + g, q1 = q0 + 8;
#pragma unroll
  for (int dt = 0; dt < 8; ++dt) {
    const int c = h * kHd + dt * 8 + 2 * t4;
    if (q0 < L)
      *reinterpret_cast<uint32_t*>(out + (seq * L + q0) * ldo + c) = pack_bf16x2(o[dt][0] * inv0, o[dt][1] * inv0);
    if (q1 < L)
      *reinterpret_cast<uint32_t*>(out + (seq * L + q1) * ldo + c) = pack_bf16x2(o[dt][2] * inv1, o[dt][3] * inv1);
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
  if (n_seq == 0) return MS_OK;
  dim3 grid((L + kBq - 1) / kBq, H, n_seq);
  launch_k(attention_kernel, grid, dim3(128), 0, st, 1, reinterpret_cast<const __nv_bfloat16*>(qkv), ld, L, H,
                                         reinterpret_cast<__nv_bfloat16*>(out), ldo, scale * 1.4426950408889634f);
  return check_launch("attention_kernel");
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
