// HBM-bound NHWC ops around the encoder GEMMs (pooling, first-layer im2col,
// global-pool + segment consensus), the op-program runner that executes a
// whole encoder forward in one native call, CUDA-event helpers for the
// profiler, and the error plumbing.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "mosel_b200.h"
#include "ptx.cuh"
#include "runtime.h"

namespace mosel {

static thread_local char g_err[512] = "";
int g_pdl = 1;

int set_error(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    char msg[256];
    snprintf(msg, sizeof msg, "%s: %s", what, cudaGetErrorString(e));
    return set_error(MS_ERR_CUDA, msg);
  }
  return MS_OK;
}

// ----------------------------------------------------------------- pooling
// one thread = one output pixel x 8 channels (16-B vectors)
__global__ void pool2d_kernel(const __nv_bfloat16* __restrict__ X, int n_img, int H, int W, int C,
                              long long xcs, int k, int stride, int pad, int OH, int OW, int is_max,
                              __nv_bfloat16* __restrict__ Y, long long ycs, int ycol0,
                              const float* __restrict__ bias, int relu) {
  pdl_trigger();
  pdl_wait();
  const int cg = C / 8;
  const long long total = (long long)n_img * OH * OW * cg;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int g = (int)(t % cg);
    long long pix = t / cg;
    const int ow = (int)(pix % OW);
    const int oh = (int)((pix / OW) % OH);
    const int n = (int)(pix / ((long long)OW * OH));
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = is_max ? -INFINITY : 0.0f;
    const int h0 = oh * stride - pad, w0 = ow * stride - pad;
    for (int dy = 0; dy < k; ++dy) {
      const int h = h0 + dy;
      if (h < 0 || h >= H) continue;
      for (int dx = 0; dx < k; ++dx) {
        const int w = w0 + dx;
        if (w < 0 || w >= W) continue;
        const uint4 v = *reinterpret_cast<const uint4*>(X + (((long long)n * H + h) * W + w) * xcs + g * 8);
        const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&v);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float f = __bfloat162float(e[j]);
          acc[j] = is_max ? fmaxf(acc[j], f) : acc[j] + f;
        }
      }
    }
    const float scale = is_max ? 1.0f : 1.0f / (float)(k * k);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float v = acc[j] * scale;
      if (bias != nullptr) v += __ldg(bias + g * 8 + j);
      if (relu) v = fmaxf(v, 0.0f);
      acc[j] = v;
    }
    uint4 o;
    o.x = pack_bf16x2(acc[0], acc[1]);
    o.y = pack_bf16x2(acc[2], acc[3]);
    o.z = pack_bf16x2(acc[4], acc[5]);
    o.w = pack_bf16x2(acc[6], acc[7]);
    *reinterpret_cast<uint4*>(Y + pix * ycs + ycol0 + g * 8) = o;
  }
}

// 3x3 pooling, row-streaming: a CTA covers TH output rows of one image; a
// thread owns one output column x 8 channels and walks down the strip,
// caching the horizontal 3-tap reduction of each input row in registers, so
// every input row is read once per column (vs 3x for a window-per-thread
// kernel).  max ignores padding; avg counts it (divide by 9).
template <bool MAX>
__device__ __forceinline__ void pool_hrow(const __nv_bfloat16* __restrict__ X, long long img, int H, int W,
                                          long long xcs, int g, int ih, int w0, float (&h)[8]) {
#pragma unroll
  for (int j = 0; j < 8; ++j) h[j] = MAX ? -INFINITY : 0.0f;
  if (ih < 0 || ih >= H) return;
#pragma unroll
  for (int dx = 0; dx < 3; ++dx) {
    const int iw = w0 + dx;
    if (iw < 0 || iw >= W) continue;
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(X + ((img * H + ih) * W + iw) * xcs + g * 8));
    const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&v);
#pragma unroll
    for (int j = 0; j < 8; ++j) h[j] = MAX ? fmaxf(h[j], __bfloat162float(e[j])) : h[j] + __bfloat162float(e[j]);
  }
}

// max pooling keeps its row state as packed bf16x2: max is exact in bf16, so
// this is bit-identical to the fp32 path with a third of the registers (more
// resident warps = more loads in flight; the kernel is latency bound)
__device__ __forceinline__ void pool_hrow_max2(const __nv_bfloat16* __restrict__ X, long long img, int H, int W,
                                               long long xcs, int g, int ih, int w0, __nv_bfloat162 (&h)[4]) {
  const __nv_bfloat162 ninf = __floats2bfloat162_rn(-INFINITY, -INFINITY);
#pragma unroll
  for (int j = 0; j < 4; ++j) h[j] = ninf;
  if (ih < 0 || ih >= H) return;
  uint4 v[3];
#pragma unroll
  for (int dx = 0; dx < 3; ++dx) {  // issue the three loads before reducing
    const int iw = w0 + dx;
    v[dx] = (iw >= 0 && iw < W) ? __ldg(reinterpret_cast<const uint4*>(X + ((img * H + ih) * W + iw) * xcs + g * 8))
                                : make_uint4(0xff80ff80u, 0xff80ff80u, 0xff80ff80u, 0xff80ff80u);
  }
#pragma unroll
  for (int dx = 0; dx < 3; ++dx) {
    const __nv_bfloat162* e = reinterpret_cast<const __nv_bfloat162*>(&v[dx]);
#pragma unroll
    for (int j = 0; j < 4; ++j) h[j] = __hmax2(h[j], e[j]);
  }
}

// 3x3 / stride 1 / pad 1 AVERAGE pooling (count_include_pad: / 9) of the
// narrow projection branches (32-128 channels), + bias + ReLU, into a channel
// slice of the block output.  A CTA stages TH+2 input rows of one frame
// (zero-padded at the borders) in shared memory with coalesced 16-B loads,
// then every output (pixel, 8 channels) is summed from shared memory in fp32.
// The register-streaming kernel spent most of its time waiting on dependent
// row loads for these tiny rows.
// 3x3 / stride 1 / pad 1 average pool (count_include_pad) + bias + ReLU,
// register-blocked: one thread = one (image, column, 8-channel group) and
// kAvgRows output rows, walking them with a rolling window of three
// horizontal 3-sums (each row's 3 loads issued together); neighbouring
// threads read neighbouring 16-B groups.  No shared memory, no barriers, and
// <= 40 registers (__launch_bounds__(256, 6)): a block fits beside a resident
// GEMM CTA (320 threads x <= 168 registers, ~200 KB smem) on the same SM, so
// the Inception pool lanes run in the issue slots the GEMMs leave idle
// instead of waiting for whole SMs.
constexpr int kAvgRows = 4;
// 4 channels (8 bytes) per thread keep the three rolling fp32 row sums in 12 registers
__device__ __forceinline__ void avg_hrow(const __nv_bfloat16* __restrict__ X, long long img, int H, int W,
                                         long long xcs, int g, int ih, int x, float (&h)[4]) {
  uint2 v[3];
#pragma unroll
  for (int dx = 0; dx < 3; ++dx) {
    const int xx = x - 1 + dx;
    v[dx] = (ih >= 0 && ih < H && xx >= 0 && xx < W)
                ? __ldg(reinterpret_cast<const uint2*>(X + ((img * H + ih) * W + xx) * xcs + g * 4))
                : make_uint2(0u, 0u);
  }
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
    for (int dx = 0; dx < 3; ++dx) {
      const float2 f = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(&v[dx])[j]);
      s2.x += f.x;
      s2.y += f.y;
    }
    h[2 * j] = s2.x;
    h[2 * j + 1] = s2.y;
  }
}
__global__ void __launch_bounds__(256, 6) avgpool3_s1_reg_kernel(const __nv_bfloat16* __restrict__ X, int n_img,
                                                                int H, int W, int C, long long xcs,
                                                                __nv_bfloat16* __restrict__ Y, long long ycs,
                                                                int ycol0, const float* __restrict__ bias, int relu) {
  pdl_trigger();
  pdl_wait();
  const int cg = C >> 2;
  const int rb_n = (H + kAvgRows - 1) / kAvgRows;
  const int total = n_img * rb_n * W * cg;  // < 2^31 (host-checked)
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int g = t % cg;
    int u = t / cg;
    const int x = u % W;
    u /= W;
    const int rb = u % rb_n;
    const long long img = u / rb_n;
    const int oh0 = rb * kAvgRows;
    float bv[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) bv[j] = bias != nullptr ? __ldg(bias + g * 4 + j) : 0.0f;
    float h0[4], h1[4], h2[4];
    avg_hrow(X, img, H, W, xcs, g, oh0 - 1, x, h0);
    avg_hrow(X, img, H, W, xcs, g, oh0, x, h1);
#pragma unroll 1
    for (int r = 0; r < kAvgRows; ++r) {
      if (oh0 + r >= H) break;
      avg_hrow(X, img, H, W, xcs, g, oh0 + r + 1, x, h2);
      uint32_t pk[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        float a = (h0[2 * j] + h1[2 * j] + h2[2 * j]) * (1.0f / 9.0f) + bv[2 * j];
        float b = (h0[2 * j + 1] + h1[2 * j + 1] + h2[2 * j + 1]) * (1.0f / 9.0f) + bv[2 * j + 1];
        if (relu) {
          a = fmaxf(a, 0.0f);
          b = fmaxf(b, 0.0f);
        }
        pk[j] = pack_bf16x2(a, b);
      }
      *reinterpret_cast<uint2*>(Y + ((img * H + oh0 + r) * W + x) * ycs + ycol0 + g * 4) = make_uint2(pk[0], pk[1]);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        h0[j] = h1[j];
        h1[j] = h2[j];
      }
    }
  }
}

constexpr int kAvgSmem = 48 * 1024;
__global__ void __launch_bounds__(256) avgpool3_s1_kernel(const __nv_bfloat16* __restrict__ X, int H, int W, int C,
                                                         long long xcs, int TH, __nv_bfloat16* __restrict__ Y,
                                                         long long ycs, int ycol0, const float* __restrict__ bias,
                                                         int relu) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ __align__(16) uint4 tile[];  // [TH+2][W+2][C/8] x 16 B
  const int cg = C / 8;
  const int wp = W + 2;
  const long long img = blockIdx.y;
  const int oh0 = blockIdx.x * TH;
  const int rows = TH + 2;
  for (int i = threadIdx.x; i < rows * wp * cg; i += blockDim.x) {
    const int g = i % cg;
    const int x = (i / cg) % wp - 1;
    const int r = i / (cg * wp);
    const int ih = oh0 - 1 + r;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (ih >= 0 && ih < H && x >= 0 && x < W)
      v = __ldg(reinterpret_cast<const uint4*>(X + ((img * H + ih) * W + x) * xcs + g * 8));
    tile[i] = v;
  }
  __syncthreads();
  const int oh1 = min(H, oh0 + TH);
  // separable box sum: vertical 3-row sums of every staged column (fp32, in
  // shared memory after the bf16 tile), then 3 horizontal neighbours per
  // output -- 2.7x fewer instructions than 9 taps per output
  float4* vsum = reinterpret_cast<float4*>(tile + rows * wp * cg);  // [TH][W+2][cg] x 8 floats (2 float4)
  for (int i = threadIdx.x; i < (oh1 - oh0) * wp * cg; i += blockDim.x) {
    const int g = i % cg;
    const int xc = (i / cg) % wp;
    const int r = i / (cg * wp);
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int dy = 0; dy < 3; ++dy) {
      const uint4 v = tile[((r + dy) * wp + xc) * cg + g];
      const __nv_bfloat162* e = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(e[j]);
        acc[2 * j] += f.x;
        acc[2 * j + 1] += f.y;
      }
    }
    vsum[2 * i] = make_float4(acc[0], acc[1], acc[2], acc[3]);
    vsum[2 * i + 1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < (oh1 - oh0) * W * cg; i += blockDim.x) {
    const int g = i % cg;
    const int x = (i / cg) % W;
    const int r = i / (cg * W);
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int dx = 0; dx < 3; ++dx) {
      const int vi = (r * wp + x + dx) * cg + g;
      const float4 a = vsum[2 * vi], b = vsum[2 * vi + 1];
      acc[0] += a.x;
      acc[1] += a.y;
      acc[2] += a.z;
      acc[3] += a.w;
      acc[4] += b.x;
      acc[5] += b.y;
      acc[6] += b.z;
      acc[7] += b.w;
    }
    uint32_t pk[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float a = acc[2 * j] * (1.0f / 9.0f), b = acc[2 * j + 1] * (1.0f / 9.0f);
      if (bias != nullptr) {
        a += bias[g * 8 + 2 * j];
        b += bias[g * 8 + 2 * j + 1];
      }
      if (relu) {
        a = fmaxf(a, 0.0f);
        b = fmaxf(b, 0.0f);
      }
      pk[j] = pack_bf16x2(a, b);
    }
    *reinterpret_cast<uint4*>(Y + ((img * H + oh0 + r) * W + x) * ycs + ycol0 + g * 8) =
        make_uint4(pk[0], pk[1], pk[2], pk[3]);
  }
}

template <int STRIDE>
__global__ void __launch_bounds__(256, 6) pool3_rows_max_kernel(const __nv_bfloat16* __restrict__ X, int H, int W,
                                                               int C, long long xcs, int pad, int OH, int OW, int TH,
                                                               __nv_bfloat16* __restrict__ Y, long long ycs,
                                                               int ycol0, const float* __restrict__ bias, int relu) {
  pdl_trigger();
  pdl_wait();
  const int cg = C / 8;
  const int t = blockIdx.z * blockDim.x + threadIdx.x;  // (column, channel group)
  if (t >= cg * OW) return;
  const int g = t % cg, ow = t / cg;
  const long long img = blockIdx.y;
  const int oh0 = blockIdx.x * TH;
  const int oh1 = min(OH, oh0 + TH);
  const int w0 = ow * STRIDE - pad;
  __nv_bfloat162 h0[4], h1[4], h2[4];
  int r0 = oh0 * STRIDE - pad;
  pool_hrow_max2(X, img, H, W, xcs, g, r0, w0, h0);
  pool_hrow_max2(X, img, H, W, xcs, g, r0 + 1, w0, h1);
  pool_hrow_max2(X, img, H, W, xcs, g, r0 + 2, w0, h2);
  for (int oh = oh0; oh < oh1; ++oh) {
    uint32_t pk[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const __nv_bfloat162 m = __hmax2(__hmax2(h0[j], h1[j]), h2[j]);
      if (bias != nullptr || relu) {
        float a = __low2float(m), b = __high2float(m);
        if (bias != nullptr) {
          a += bias[g * 8 + 2 * j];
          b += bias[g * 8 + 2 * j + 1];
        }
        if (relu) {
          a = fmaxf(a, 0.0f);
          b = fmaxf(b, 0.0f);
        }
        pk[j] = pack_bf16x2(a, b);
      } else {
        pk[j] = *reinterpret_cast<const uint32_t*>(&m);
      }
    }
    *reinterpret_cast<uint4*>(Y + ((img * OH + oh) * OW + ow) * ycs + ycol0 + g * 8) =
        make_uint4(pk[0], pk[1], pk[2], pk[3]);
    if (oh + 1 < oh1) {
      r0 += STRIDE;
      if (STRIDE == 1) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          h0[j] = h1[j];
          h1[j] = h2[j];
        }
        pool_hrow_max2(X, img, H, W, xcs, g, r0 + 2, w0, h2);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) h0[j] = h2[j];
        pool_hrow_max2(X, img, H, W, xcs, g, r0 + 1, w0, h1);
        pool_hrow_max2(X, img, H, W, xcs, g, r0 + 2, w0, h2);
      }
    }
  }
}

template <bool MAX, int STRIDE>
__global__ void __launch_bounds__(512) pool3_rows_kernel(const __nv_bfloat16* __restrict__ X, int H, int W, int C, long long xcs,
                                  int pad, int OH, int OW, int TH, __nv_bfloat16* __restrict__ Y,
                                  long long ycs, int ycol0, const float* __restrict__ bias, int relu) {
  pdl_trigger();
  pdl_wait();
  const int cg = C / 8;
  const int t = blockIdx.z * blockDim.x + threadIdx.x;  // (column, channel group)
  if (t >= cg * OW) return;
  const int g = t % cg, ow = t / cg;
  const long long img = blockIdx.y;
  const int oh0 = blockIdx.x * TH;
  const int oh1 = min(OH, oh0 + TH);
  const int w0 = ow * STRIDE - pad;
  float bsum[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) bsum[j] = (bias != nullptr) ? bias[g * 8 + j] : 0.0f;
  // rows r0, r0+1, r0+2 of the current output row, reduced horizontally
  float h0[8], h1[8], h2[8];
  int r0 = oh0 * STRIDE - pad;
  pool_hrow<MAX>(X, img, H, W, xcs, g, r0, w0, h0);
  pool_hrow<MAX>(X, img, H, W, xcs, g, r0 + 1, w0, h1);
  pool_hrow<MAX>(X, img, H, W, xcs, g, r0 + 2, w0, h2);
  for (int oh = oh0; oh < oh1; ++oh) {
    uint32_t pk[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float a, b;
      if (MAX) {
        a = fmaxf(fmaxf(h0[2 * j], h1[2 * j]), h2[2 * j]);
        b = fmaxf(fmaxf(h0[2 * j + 1], h1[2 * j + 1]), h2[2 * j + 1]);
      } else {
        a = (h0[2 * j] + h1[2 * j] + h2[2 * j]) * (1.0f / 9.0f);
        b = (h0[2 * j + 1] + h1[2 * j + 1] + h2[2 * j + 1]) * (1.0f / 9.0f);
      }
      a += bsum[2 * j];
      b += bsum[2 * j + 1];
      if (relu) {
        a = fmaxf(a, 0.0f);
        b = fmaxf(b, 0.0f);
      }
      pk[j] = pack_bf16x2(a, b);
    }
    *reinterpret_cast<uint4*>(Y + ((img * OH + oh) * OW + ow) * ycs + ycol0 + g * 8) =
        make_uint4(pk[0], pk[1], pk[2], pk[3]);
    if (oh + 1 < oh1) {
      r0 += STRIDE;
      if (STRIDE == 1) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          h0[j] = h1[j];
          h1[j] = h2[j];
        }
        pool_hrow<MAX>(X, img, H, W, xcs, g, r0 + 2, w0, h2);
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) h0[j] = h2[j];
        pool_hrow<MAX>(X, img, H, W, xcs, g, r0 + 1, w0, h1);
        pool_hrow<MAX>(X, img, H, W, xcs, g, r0 + 2, w0, h2);
      }
    }
  }
}

static int pool_out(int in, int k, int stride, int pad, int ceil_mode) {
  const int span = in + 2 * pad - k;
  int o = (ceil_mode ? (span + stride - 1) / stride : span / stride) + 1;
  // a window must start inside the (left-padded) input
  if (ceil_mode && (o - 1) * stride >= in + pad) --o;
  return o;
}

// -------------------------------------------------------------- im2col
// One thread = one output pixel x 8 consecutive K columns (one 16-B store,
// coalesced across threads).  K index = (kh*KW + kw)*C + c; the 8 source
// elements are scalar loads that hit L1/L2 (each input element is reused by
// ~KH*KW/stride^2 overlapping windows).
__global__ void im2col_kernel(const __nv_bfloat16* __restrict__ X, int n_img, int H, int W, int C, int KH,
                              int KW, int stride, int pad, int OH, int OW, __nv_bfloat16* __restrict__ out,
                              int K_pad) {
  pdl_trigger();
  pdl_wait();
  const int k8n = K_pad / 8;
  const long long total = (long long)n_img * OH * OW * k8n;
  const int kreal = KH * KW * C;
  const unsigned short* Xs = reinterpret_cast<const unsigned short*>(X);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int k8 = (int)(t % k8n);
    const long long pix = t / k8n;
    const int ow = (int)(pix % OW);
    const int oh = (int)((pix / OW) % OH);
    const int n = (int)(pix / ((long long)OW * OH));
    const long long img = (long long)n * H * W;
    int k = k8 * 8;
    int c = k % C;
    int tap = k / C;
    int kw = tap % KW, kh = tap / KW;
    unsigned short v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      unsigned short e = 0;
      if (k + j < kreal) {
        const int h = oh * stride - pad + kh, w = ow * stride - pad + kw;
        if (h >= 0 && h < H && w >= 0 && w < W) e = __ldg(Xs + (img + (long long)h * W + w) * C + c);
      }
      v[j] = e;
      if (++c == C) {
        c = 0;
        if (++kw == KW) {
          kw = 0;
          ++kh;
        }
      }
    }
    uint4 o;
    o.x = v[0] | ((unsigned)v[1] << 16);
    o.y = v[2] | ((unsigned)v[3] << 16);
    o.z = v[4] | ((unsigned)v[5] << 16);
    o.w = v[6] | ((unsigned)v[7] << 16);
    reinterpret_cast<uint4*>(out)[t] = o;
  }
}

// ----------------------------------------- global pool + segment consensus
// Y[r, c] = mean over the S*HW pixels of request r's S frames.  One CTA per
// (request, 32 channel groups = 256 channels); its 256 threads are 32 channel
// groups x 8 pixel slices (each warp reads 512 contiguous bytes per row),
// reduced through shared memory.
constexpr int kSegSlices = 8;
__global__ void __launch_bounds__(256) segment_mean_kernel(const __nv_bfloat16* __restrict__ X, int n_req, int S,
                                                           int HW, int C, __nv_bfloat16* __restrict__ Y,
                                                           long long y_ld) {
  pdl_trigger();
  pdl_wait();
  __shared__ float part[kSegSlices][32][9];
  const int cg = C / 8;
  const int lane = threadIdx.x & 31, slice = threadIdx.x >> 5;
  const int g = blockIdx.y * 32 + lane;
  const long long r = blockIdx.x;
  const long long rows = (long long)S * HW;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (g < cg) {
    const __nv_bfloat16* base = X + r * rows * C + g * 8;
    for (long long p = slice; p < rows; p += kSegSlices) {
      const uint4 v = *reinterpret_cast<const uint4*>(base + p * C);
      const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&v);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += __bfloat162float(e[j]);
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) part[slice][lane][j] = acc[j];
  __syncthreads();
  if (slice == 0 && g < cg) {
    float t[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) t[j] = 0.0f;
    // fixed summation order (slice 0..7) keeps the result deterministic
    for (int q = 0; q < kSegSlices; ++q)
#pragma unroll
      for (int j = 0; j < 8; ++j) t[j] += part[q][lane][j];
    const float s = 1.0f / (float)rows;
    uint4 o;
    o.x = pack_bf16x2(t[0] * s, t[1] * s);
    o.y = pack_bf16x2(t[2] * s, t[3] * s);
    o.z = pack_bf16x2(t[4] * s, t[5] * s);
    o.w = pack_bf16x2(t[6] * s, t[7] * s);
    *reinterpret_cast<uint4*>(Y + r * y_ld + g * 8) = o;
  }
}

static int grid_for(long long work, int threads) {
  long long b = (work + threads - 1) / threads;
  const long long cap = 148LL * 32;  // grid-stride beyond 32 CTAs per SM
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

// ---------------------------------------------------------- op programs
enum OpKind : int {
  OP_GEMM = 1, OP_POOL = 2, OP_IM2COL = 3, OP_SEGMEAN = 4,
  OP_LAYERNORM = 5, OP_ATTENTION = 6, OP_PATCHIFY = 7, OP_VIT_EMBED = 8, OP_BERT_EMBED = 9
};

struct PoolArgs {
  const void* X;
  void* Y;
  long long xcs, ycs;
  int n_img, H, W, C, k, stride, pad, ceil_mode, is_max, ycol0;
  const float* bias;
  int relu;
};
struct Im2colArgs {
  const void* X;
  void* out;
  int n_img, H, W, C, KH, KW, stride, pad, K_pad;
};
struct SegArgs {
  const void* X;
  void* Y;
  long long y_ld;
  int n_req, S, HW, C;
};

struct LnArgs {
  const void* X;
  void* Y;
  const float *gamma, *beta;
  long long ldx, rows, ldy;
  int C;
  float eps;
};
struct AttnArgs {
  const void* qkv;
  void* out;
  long long ld, ldo;
  int L, H, n_seq;
  float scale;
};
struct PatchArgs {
  const void* X;
  void* Y;
  int n, S, C, P;
};
struct VitEmbedArgs {
  const void *pe, *cls, *pos;
  void* tok;
  int n, L, D;
};
struct BertEmbedArgs {
  const int32_t* ids;
  const void *word, *pos, *type0;
  const float *gamma, *beta;
  void* Y;
  long long n_tok;
  int L, D;
  float eps;
};

struct alignas(64) Op {
  int kind;
  int pad_[15];
  union {
    unsigned char plan[MS_GEMM_PLAN_BYTES];
    PoolArgs pool;
    Im2colArgs im2col;
    SegArgs seg;
    LnArgs ln;
    AttnArgs attn;
    PatchArgs patch;
    VitEmbedArgs vit;
    BertEmbedArgs bert;
  } u;
};
static_assert(sizeof(Op) <= MS_OP_BYTES && MS_OP_BYTES % 64 == 0, "MS_OP_BYTES too small / misaligned");

static int run_pool(const PoolArgs& a, cudaStream_t st) {
  if (a.C % 8 != 0 || a.xcs % 8 != 0 || a.ycs % 8 != 0 || a.ycol0 % 8 != 0)
    return set_error(MS_ERR_INVALID, "pool2d needs channel counts/strides multiple of 8");
  const int OH = pool_out(a.H, a.k, a.stride, a.pad, a.ceil_mode);
  const int OW = pool_out(a.W, a.k, a.stride, a.pad, a.ceil_mode);
  const int threads = (a.C / 8) * OW;
  static const bool avg_smem = getenv("MS_AVGPOOL_SMEM") != nullptr;  // A/B: the smem-staged kernel
  if (!a.is_max && a.k == 3 && a.stride == 1 && a.pad == 1 && !avg_smem) {
    const long long items = (long long)a.n_img * ((a.H + kAvgRows - 1) / kAvgRows) * a.W * (a.C / 4);
    if (items >= (1LL << 31)) return set_error(MS_ERR_INVALID, "avg pool: too many work items");
    long long blocks = (items + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    launch_k(avgpool3_s1_reg_kernel, dim3((unsigned)blocks), dim3(256), 0, st, 1,
             reinterpret_cast<const __nv_bfloat16*>(a.X), a.n_img, a.H, a.W, a.C, a.xcs,
             reinterpret_cast<__nv_bfloat16*>(a.Y), a.ycs, a.ycol0, a.bias, a.relu);
    return check_launch("avgpool3_s1_reg_kernel");
  }
  if (!a.is_max && a.k == 3 && a.stride == 1 && a.pad == 1 && a.n_img <= 65535 &&
      5 * (a.W + 2) * a.C * 2 <= kAvgSmem) {
    // the fp32 sums of 9 taps: order per output (dy, dx) = the oracle's window order up to fp32 rounding
    const int row_bytes = (a.W + 2) * a.C * 2;  // bf16 staged row; its fp32 vertical sums take 2x
    int TH = (kAvgSmem - 2 * row_bytes) / (3 * row_bytes);
    if (TH > a.H) TH = a.H;
    if (TH < 1) TH = 1;
    dim3 grid((a.H + TH - 1) / TH, a.n_img);
    const size_t smem = (size_t)(TH + 2) * row_bytes + (size_t)TH * row_bytes * 2;
    launch_k(avgpool3_s1_kernel, grid, dim3(256), smem, st, 1, reinterpret_cast<const __nv_bfloat16*>(a.X), a.H,
             a.W, a.C, a.xcs, TH, reinterpret_cast<__nv_bfloat16*>(a.Y), a.ycs, a.ycol0, a.bias, a.relu);
    return check_launch("avgpool3_s1_kernel");
  }
  if (a.k == 3 && (a.stride == 1 || a.stride == 2) && a.n_img <= 65535) {
    // <= 256 threads x <= 40 registers: max-pool blocks fit beside a resident
    // GEMM CTA (see avgpool3_s1_reg_kernel); the other pool kernels keep 512
    const int cap = a.is_max ? 256 : 512;
    const int block = threads < cap ? (threads + 31) / 32 * 32 : cap;
    // output rows per thread: the largest of 8/4/2/1 whose grid fills its
    // last wave of resident blocks to >= 85% (a 1.1-wave grid idles half the
    // GPU in its tail); fewer rows cost only L2 re-reads of window rows
    const int gz = (threads + block - 1) / block;
    const int resident = 148 * (2048 / block);
    int TH = 8;
    for (int th = 8; th >= 1; th >>= 1) {
      const long long blocks = (long long)((OH + th - 1) / th) * a.n_img * gz;
      const double waves = (double)blocks / resident;
      TH = th;
      if (waves / ceil(waves) >= 0.85) break;
    }
    dim3 grid((OH + TH - 1) / TH, a.n_img, gz);
    auto X = reinterpret_cast<const __nv_bfloat16*>(a.X);
    auto Y = reinterpret_cast<__nv_bfloat16*>(a.Y);
    if (a.is_max && a.stride == 2)
      launch_k(pool3_rows_max_kernel<2>, grid, dim3(block), 0, st, 1, X, a.H, a.W, a.C, a.xcs, a.pad, OH, OW, TH, Y,
               a.ycs, a.ycol0, a.bias, a.relu);
    else if (a.is_max)
      launch_k(pool3_rows_max_kernel<1>, grid, dim3(block), 0, st, 1, X, a.H, a.W, a.C, a.xcs, a.pad, OH, OW, TH, Y,
               a.ycs, a.ycol0, a.bias, a.relu);
    else if (a.stride == 2)
      launch_k(pool3_rows_kernel<false, 2>, grid, dim3(block), 0, st, 1, X, a.H, a.W, a.C, a.xcs, a.pad, OH, OW, TH, Y, a.ycs,
                                                         a.ycol0, a.bias, a.relu);
    else
      launch_k(pool3_rows_kernel<false, 1>, grid, dim3(block), 0, st, 1, X, a.H, a.W, a.C, a.xcs, a.pad, OH, OW, TH, Y, a.ycs,
                                                         a.ycol0, a.bias, a.relu);
    return check_launch("pool3_rows_kernel");
  }
  const long long work = (long long)a.n_img * OH * OW * (a.C / 8);
  launch_k(pool2d_kernel, dim3(grid_for(work, 256)), dim3(256), 0, st, 1,
      reinterpret_cast<const __nv_bfloat16*>(a.X), a.n_img, a.H, a.W, a.C, a.xcs, a.k, a.stride, a.pad, OH, OW,
      a.is_max, reinterpret_cast<__nv_bfloat16*>(a.Y), a.ycs, a.ycol0, a.bias, a.relu);
  return check_launch("pool2d_kernel");
}

static int run_im2col(const Im2colArgs& a, cudaStream_t st) {
  const int OH = (a.H + 2 * a.pad - a.KH) / a.stride + 1;
  const int OW = (a.W + 2 * a.pad - a.KW) / a.stride + 1;
  if (a.K_pad % 8 != 0) return set_error(MS_ERR_INVALID, "im2col K_pad must be a multiple of 8");
  const long long work = (long long)a.n_img * OH * OW * (a.K_pad / 8);
  launch_k(im2col_kernel, dim3(grid_for(work, 256)), dim3(256), 0, st, 1, reinterpret_cast<const __nv_bfloat16*>(a.X), a.n_img, a.H,
                                                      a.W, a.C, a.KH, a.KW, a.stride, a.pad, OH, OW,
                                                      reinterpret_cast<__nv_bfloat16*>(a.out), a.K_pad);
  return check_launch("im2col_kernel");
}

static int run_segmean(const SegArgs& a, cudaStream_t st) {
  if (a.C % 8 != 0 || a.y_ld % 8 != 0) return set_error(MS_ERR_INVALID, "segment_mean needs C % 8 == 0");
  if (a.n_req <= 0) return MS_OK;
  const dim3 grid((unsigned)a.n_req, (unsigned)((a.C / 8 + 31) / 32));
  launch_k(segment_mean_kernel, grid, dim3(256), 0, st, 1, reinterpret_cast<const __nv_bfloat16*>(a.X), a.n_req,
                                                            a.S, a.HW, a.C, reinterpret_cast<__nv_bfloat16*>(a.Y),
                                                            a.y_ld);
  return check_launch("segment_mean_kernel");
}

}  // namespace mosel

using namespace mosel;

extern "C" {

int ms_abi_version(void) { return 4; }
int ms_set_pdl(int enable) {
  const int prev = g_pdl;
  g_pdl = enable ? 1 : 0;
  return prev;
}
const char* ms_last_error(void) { return g_err; }
int ms_device_sync(void) {
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return set_error(MS_ERR_CUDA, cudaGetErrorString(e));
  return MS_OK;
}

int ms_pool2d(const void* X, int n_img, int H, int W, int C, long long x_cstride, int k, int stride, int pad,
              int ceil_mode, int is_max, void* Y, long long y_cstride, int y_col0, void* stream) {
  PoolArgs a{X, Y, x_cstride, y_cstride, n_img, H, W, C, k, stride, pad, ceil_mode, is_max, y_col0, nullptr, 0};
  return run_pool(a, reinterpret_cast<cudaStream_t>(stream));
}

int ms_pool2d_ex(const void* X, int n_img, int H, int W, int C, long long x_cstride, int k, int stride, int pad,
                 int ceil_mode, int is_max, void* Y, long long y_cstride, int y_col0, const float* bias, int relu,
                 void* stream) {
  PoolArgs a{X, Y, x_cstride, y_cstride, n_img, H, W, C, k, stride, pad, ceil_mode, is_max, y_col0, bias, relu};
  return run_pool(a, reinterpret_cast<cudaStream_t>(stream));
}

int ms_im2col(const void* X, int n_img, int H, int W, int C, int KH, int KW, int stride, int pad, void* out,
              int K_pad, void* stream) {
  Im2colArgs a{X, out, n_img, H, W, C, KH, KW, stride, pad, K_pad};
  return run_im2col(a, reinterpret_cast<cudaStream_t>(stream));
}

int ms_segment_mean(const void* X, int n_req, int S, int HW, int C, void* Y, long long y_ld, void* stream) {
  SegArgs a{X, Y, y_ld, n_req, S, HW, C};
  return run_segmean(a, reinterpret_cast<cudaStream_t>(stream));
}

int ms_op_gemm(void* op, const void* plan) {
  if (!op || !plan) return set_error(MS_ERR_INVALID, "null op/plan");
  Op* o = reinterpret_cast<Op*>(op);
  memset(o, 0, sizeof(Op));
  o->kind = OP_GEMM;
  memcpy(o->u.plan, plan, MS_GEMM_PLAN_BYTES);
  return MS_OK;
}

int ms_op_pool2d(void* op, const void* X, int n_img, int H, int W, int C, long long x_cstride, int k, int stride,
                 int pad, int ceil_mode, int is_max, void* Y, long long y_cstride, int y_col0) {
  if (!op) return set_error(MS_ERR_INVALID, "null op");
  Op* o = reinterpret_cast<Op*>(op);
  memset(o, 0, sizeof(Op));
  o->kind = OP_POOL;
  o->u.pool = PoolArgs{X, Y, x_cstride, y_cstride, n_img, H, W, C, k, stride, pad, ceil_mode, is_max, y_col0,
                       nullptr, 0};
  return MS_OK;
}

int ms_op_pool2d_ex(void* op, const void* X, int n_img, int H, int W, int C, long long x_cstride, int k, int stride,
                    int pad, int ceil_mode, int is_max, void* Y, long long y_cstride, int y_col0, const float* bias,
                    int relu) {
  int rc = ms_op_pool2d(op, X, n_img, H, W, C, x_cstride, k, stride, pad, ceil_mode, is_max, Y, y_cstride, y_col0);
  if (rc) return rc;
  Op* o = reinterpret_cast<Op*>(op);
  o->u.pool.bias = bias;
  o->u.pool.relu = relu;
  return MS_OK;
}

int ms_op_im2col(void* op, const void* X, int n_img, int H, int W, int C, int KH, int KW, int stride, int pad,
                 void* out, int K_pad) {
  if (!op) return set_error(MS_ERR_INVALID, "null op");
  Op* o = reinterpret_cast<Op*>(op);
  memset(o, 0, sizeof(Op));
  o->kind = OP_IM2COL;
  o->u.im2col = Im2colArgs{X, out, n_img, H, W, C, KH, KW, stride, pad, K_pad};
  return MS_OK;
}

int ms_op_segment_mean(void* op, const void* X, int n_req, int S, int HW, int C, void* Y, long long y_ld) {
  if (!op) return set_error(MS_ERR_INVALID, "null op");
  Op* o = reinterpret_cast<Op*>(op);
  memset(o, 0, sizeof(Op));
  o->kind = OP_SEGMEAN;
  o->u.seg = SegArgs{X, Y, y_ld, n_req, S, HW, C};
  return MS_OK;
}

static Op* op_reset(void* op, int kind) {
  Op* o = reinterpret_cast<Op*>(op);
  memset(o, 0, sizeof(Op));
  o->kind = kind;
  return o;
}

int ms_op_layernorm(void* op, const void* X, long long ldx, long long rows, const float* gamma, const float* beta,
                    void* Y, long long ldy, int C, float eps) {
  if (!op) return set_error(MS_ERR_INVALID, "null op");
  op_reset(op, OP_LAYERNORM)->u.ln = LnArgs{X, Y, gamma, beta, ldx, rows, ldy, C, eps};
  return MS_OK;
}

int ms_op_attention(void* op, const void* qkv, long long ld, int L, int H, int n_seq, void* out, long long ldo,
                    float scale) {
  if (!op) return set_error(MS_ERR_INVALID, "null op");
  op_reset(op, OP_ATTENTION)->u.attn = AttnArgs{qkv, out, ld, ldo, L, H, n_seq, scale};
  return MS_OK;
}

int ms_op_patchify(void* op, const void* X, int n, int S, int C, int P, void* Y) {
  if (!op) return set_error(MS_ERR_INVALID, "null op");
  op_reset(op, OP_PATCHIFY)->u.patch = PatchArgs{X, Y, n, S, C, P};
  return MS_OK;
}

int ms_op_vit_embed(void* op, const void* pe, const void* cls, const void* pos, int n, int L, int D, void* tok) {
  if (!op) return set_error(MS_ERR_INVALID, "null op");
  op_reset(op, OP_VIT_EMBED)->u.vit = VitEmbedArgs{pe, cls, pos, tok, n, L, D};
  return MS_OK;
}

int ms_op_bert_embed(void* op, const int32_t* ids, long long n_tok, int L, const void* word, const void* pos,
                     const void* type0, const float* gamma, const float* beta, void* Y, int D, float eps) {
  if (!op) return set_error(MS_ERR_INVALID, "null op");
  op_reset(op, OP_BERT_EMBED)->u.bert = BertEmbedArgs{ids, word, pos, type0, gamma, beta, Y, n_tok, L, D, eps};
  return MS_OK;
}

int ms_program_run(const void* ops, int n_ops, void* stream) {
  const unsigned char* base = reinterpret_cast<const unsigned char*>(ops);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  for (int i = 0; i < n_ops; ++i) {
    // ops are laid out MS_OP_BYTES apart (the ABI stride), not sizeof(Op)
    const Op& o = *reinterpret_cast<const Op*>(base + (size_t)i * MS_OP_BYTES);
    int rc = MS_OK;
    switch (o.kind) {
      case OP_GEMM: rc = ms_gemm_run(o.u.plan, stream); break;
      case OP_POOL: rc = run_pool(o.u.pool, st); break;
      case OP_IM2COL: rc = run_im2col(o.u.im2col, st); break;
      case OP_SEGMEAN: rc = run_segmean(o.u.seg, st); break;
      case OP_LAYERNORM: {
        const LnArgs& a = o.u.ln;
        rc = run_layernorm(a.X, a.ldx, a.rows, a.gamma, a.beta, a.Y, a.ldy, a.C, a.eps, st);
        break;
      }
      case OP_ATTENTION: {
        const AttnArgs& a = o.u.attn;
        rc = run_attention(a.qkv, a.ld, a.L, a.H, a.n_seq, a.out, a.ldo, a.scale, st);
        break;
      }
      case OP_PATCHIFY: rc = run_patchify(o.u.patch.X, o.u.patch.n, o.u.patch.S, o.u.patch.C, o.u.patch.P, o.u.patch.Y, st); break;
      case OP_VIT_EMBED: {
        const VitEmbedArgs& a = o.u.vit;
        rc = run_vit_embed(a.pe, a.cls, a.pos, a.n, a.L, a.D, a.tok, st);
        break;
      }
      case OP_BERT_EMBED: {
        const BertEmbedArgs& a = o.u.bert;
        rc = run_bert_embed(a.ids, a.n_tok, a.L, a.word, a.pos, a.type0, a.gamma, a.beta, a.Y, a.D, a.eps, st);
        break;
      }
      default: rc = set_error(MS_ERR_INVALID, "unknown op kind");
    }
    if (rc != MS_OK) return rc;
  }
  return MS_OK;
}

int ms_event_create(void** ev) {
  cudaEvent_t e;
  if (cudaEventCreate(&e) != cudaSuccess) return set_error(MS_ERR_CUDA, "cudaEventCreate failed");
  *ev = reinterpret_cast<void*>(e);
  return MS_OK;
}
int ms_event_destroy(void* ev) {
  cudaEventDestroy(reinterpret_cast<cudaEvent_t>(ev));
  return MS_OK;
}
int ms_event_record(void* ev, void* stream) {
  if (cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev), reinterpret_cast<cudaStream_t>(stream)) != cudaSuccess)
    return set_error(MS_ERR_CUDA, "cudaEventRecord failed");
  return MS_OK;
}
int ms_event_query(void* ev) {
  cudaError_t e = cudaEventQuery(reinterpret_cast<cudaEvent_t>(ev));
  if (e == cudaSuccess) return 0;
  if (e == cudaErrorNotReady) return 1;
  set_error(MS_ERR_CUDA, cudaGetErrorString(e));
  return -1;
}

int ms_stream_wait_event(void* stream, void* ev) {
  if (cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(stream), reinterpret_cast<cudaEvent_t>(ev), 0) != cudaSuccess)
    return set_error(MS_ERR_CUDA, "cudaStreamWaitEvent failed");
  return MS_OK;
}
int ms_graph_launch(void* graph_exec, void* stream) {
  if (cudaGraphLaunch(reinterpret_cast<cudaGraphExec_t>(graph_exec), reinterpret_cast<cudaStream_t>(stream)) !=
      cudaSuccess)
    return set_error(MS_ERR_CUDA, "cudaGraphLaunch failed");
  return MS_OK;
}

int ms_event_elapsed_us(void* start, void* stop, double* us) {
  float ms = 0.0f;
  if (cudaEventSynchronize(reinterpret_cast<cudaEvent_t>(stop)) != cudaSuccess ||
      cudaEventElapsedTime(&ms, reinterpret_cast<cudaEvent_t>(start), reinterpret_cast<cudaEvent_t>(stop)) !=
          cudaSuccess)
    return set_error(MS_ERR_CUDA, "cudaEventElapsedTime failed");
  *us = 1000.0 * (double)ms;
  return MS_OK;
}

}  // extern "C"
