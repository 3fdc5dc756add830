// Fused 3x3 / stride-1 / pad-1 convolution + bias + ReLU + 3x3 / stride-2
// ceil-mode max pool (BN-Inception conv2 -> pool2 at 56x56 -> 28x28).
//
// The unfused pair writes the 56^2 x 192 conv map (4x the pooled bytes) and
// reads it back in a separate pool kernel; here the pooled rows leave the
// epilogue registers directly.
//
// Tiles are the halo tiles of MODE_CONV_HALO with P = 64 (ceil8(W + 2), so
// bh = 2 conv rows per 128-row M tile): M row m = y * 64 + x.  Per 64-channel
// chunk ONE TMA box brings the 4 x 64 halo of input pixels (zero fill at the
// borders), the 9 taps are MMAs on views shifted by (dy * 64 + dx) rows, and
// the weights stream per tap (the 9 x 64 x N weight blocks do not fit beside
// the halos).
//
// Work: a CTA owns a contiguous range of pooled rows (image, i).  Pooled row i
// needs conv rows 2i, 2i+1, 2i+2, and consecutive pooled rows share conv row
// 2i+2, so the walk is one tile per pooled row -- CLOSE(i) = conv rows
// (2i+1, 2i+2) -- preceded by OPEN(i) = conv rows (2i-1, 2i) where a run
// starts (the range's first row or an image's first row; only its second
// row is used).  StemWalk (gemm_plan.h) is the same walk as the fused stem's.
//
// Epilogue (8 warps = 2 channel groups x 4 TMEM lane quarters): lane quarter
// q holds conv row y = q / 2 at x = 32 (q & 1) + lane.  The y = 1 warps keep
// conv row 2i (carried from the previous tile) and row 2i+2 in registers; the
// y = 0 warps pass row 2i+1 through a padded shared-memory row; the vertical
// max is a register max, the horizontal 3-max two warp shuffles (the one
// window that crosses the x = 32 warp boundary reads the neighbour warp's
// value from shared memory).  bf16 rounding, bias and ReLU commute with max,
// so Y == maxpool(bf16(relu(conv + bias))) bit for bit -- the unfused halo
// conv + pool pair accumulates in the same (chunk, tap, k) order.
#include <cstdio>

#include "gemm_plan.h"
#include "ptx.cuh"
#include "runtime.h"

namespace mosel {

namespace {

constexpr int kCPThreads = 64 + 32 * kEpiWarps;
constexpr int kCPPitch = 64;                // halo row width (pixels)
constexpr int kCPHaloRows = 4;              // bh + 2
constexpr int kXRowBytesMax = 4 * 64 + 16;  // one pixel's channels of a group (<= 128 ch) + 16-B pad

__device__ __forceinline__ uint32_t bmax2(uint32_t a, uint32_t b) {
  __nv_bfloat162 r = __hmax2(*reinterpret_cast<__nv_bfloat162*>(&a), *reinterpret_cast<__nv_bfloat162*>(&b));
  return *reinterpret_cast<uint32_t*>(&r);
}

struct PoolWalk {  // conv rows: OPEN -> {2i} (tile rows 2i-1, 2i); CLOSE -> {2i+1, 2i+2 < OH}
  int u, u1, PH, OH, img, i;
  bool open;
  __device__ __forceinline__ void begin(int u0_, int u1_, int PH_, int OH_) {
    u1 = u1_; PH = PH_; OH = OH_; u = u0_;
    img = u / PH;
    i = u - img * PH;
    open = true;
  }
  __device__ __forceinline__ bool valid() const { return u < u1; }
  __device__ __forceinline__ void next() {
    if (open) { open = false; return; }
    ++u;
    if (++i == PH) {
      i = 0;
      ++img;
      open = true;
    }
  }
  __device__ __forceinline__ int tile_row0() const { return open ? 2 * i - 1 : 2 * i + 1; }
  __device__ __forceinline__ bool second_row() const { return open || 2 * i + 2 < OH; }
};

// CPG: 32-channel chunks per epilogue group (N = 64 * CPG output channels).
// kHalo: halo tiles (W 55..62, pitch 64); else (W == 64) tap boxes: per
// (chunk, tap) one {64 ch, 64 px, 2 rows} TMA box at the tap-shifted
// coordinate beside the weights in each pipeline stage (OOB zero fill = the
// padding) -- the same M-row mapping y * 64 + x, every column real.
template <int CPG, bool kHalo>
__global__ void __launch_bounds__(kCPThreads, 1)
    conv_pool_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ GemmParams p) {
  constexpr int N = 64 * CPG;
  constexpr int kXRow = CPG * 64 + 16;  // bytes per pixel row of the exchange buffer (16-B pad: no bank conflicts)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
  const int stages = p.stages;
  uint8_t* smA = smem;                                   // 2 halo slots | tap-box A ring
  uint8_t* smB = smA + (kHalo ? 2 * p.halo_slot : stages * kABytes);  // weight ring
  uint8_t* xbuf = smB + stages * p.b_bytes;              // [2 groups][64 px][kXRow]
  uint32_t* bnd = reinterpret_cast<uint32_t*>(xbuf + 2 * 64 * kXRow);  // [2 groups][CPG * 16]
  uint64_t* full = reinterpret_cast<uint64_t*>(bnd + 2 * CPG * 16);
  uint64_t* empty = full + stages;
  uint64_t* afull = empty + stages;
  uint64_t* aempty = afull + 2;
  uint64_t* tfull = aempty + 2;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* sbias = reinterpret_cast<float*>(tmem_slot + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int u0 = (int)((long long)p.units * blockIdx.x / gridDim.x);
  const int u1 = (int)((long long)p.units * (blockIdx.x + 1) / gridDim.x);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&afull[a], 1);
      mbar_init(&aempty[a], 1);
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  for (int c = threadIdx.x; c < N; c += blockDim.x) sbias[c] = p.bias ? p.bias[c] : 0.0f;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_trigger();  // after the TMEM allocation (see gemm_tc_kernel)
  pdl_wait();

  PoolWalk w;
  w.begin(u0, u1, p.PH, p.OH);
  if (warp == 0) {
    if (lane == 0) {  // ----------------------------------------- TMA producer
      int s = 0, hs = 0;
      uint32_t phase = 0, hphase = 0;
      for (; w.valid() && !kHalo; w.next()) {
        for (int cc = 0; cc < p.cchunks; ++cc) {
          for (int tap = 0; tap < 9; ++tap) {
            const int dy = tap / 3, dx = tap - 3 * (tap / 3);
            mbar_wait(&empty[s], phase ^ 1);
            mbar_arrive_expect_tx(&full[s], kABytes + p.b_bytes);
            tma_load_4d(smem_addr(smA + s * kABytes), &tmA, &full[s], cc * kBK, dx - 1, w.tile_row0() + dy - 1, w.img);
            tma_load_2d(smem_addr(smB + s * p.b_bytes), &tmB, &full[s], (tap * p.cchunks + cc) * kBK, 0);
            if (++s == stages) {
              s = 0;
              phase ^= 1;
            }
          }
        }
      }
      for (; w.valid() && kHalo; w.next()) {
        for (int cc = 0; cc < p.cchunks; ++cc) {
          mbar_wait(&aempty[hs], hphase ^ 1);
          mbar_arrive_expect_tx(&afull[hs], p.a_bytes);
          tma_load_4d(smem_addr(smA + hs * p.halo_slot), &tmA, &afull[hs], cc * kBK, -1, w.tile_row0() - 1, w.img);
          for (int tap = 0; tap < 9; ++tap) {
            mbar_wait(&empty[s], phase ^ 1);
            mbar_arrive_expect_tx(&full[s], p.b_bytes);
            tma_load_2d(smem_addr(smB + s * p.b_bytes), &tmB, &full[s], (tap * p.cchunks + cc) * kBK, 0);
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
    }
  } else if (warp == 1) {  // ------------------------------------ MMA issuer
    const uint32_t idesc = umma_idesc_bf16_m128((uint32_t)N);
    int s = 0, hs = 0;
    uint32_t phase = 0, hphase = 0;
    for (int k = 0; w.valid(); w.next(), ++k) {
      const int slot = k & 1;
      mbar_wait(&tempty[slot], (uint32_t)(((k >> 1) & 1) ^ 1));
      tc_fence_after();
      const uint32_t d = tmem_base + (uint32_t)(slot * 256);
      for (int cc = 0; cc < p.cchunks; ++cc) {
        if (kHalo) {
          mbar_wait(&afull[hs], hphase);
          tc_fence_after();
        }
        const uint32_t halo = smem_addr(smA + hs * p.halo_slot);
        for (int tap = 0; tap < 9; ++tap) {
          mbar_wait(&full[s], phase);
          tc_fence_after();
          if (lane == 0) {
            const int dy = tap / 3, dx = tap - 3 * (tap / 3);
            const uint64_t adesc = kHalo ? umma_desc_sw128(halo + (uint32_t)((dy * kCPPitch + dx) * 128))
                                         : umma_desc_sw128(smem_addr(smA + s * kABytes));
            const uint64_t bdesc = umma_desc_sw128(smem_addr(smB + s * p.b_bytes));
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk)
              umma_bf16(d, adesc + 2 * kk, bdesc + 2 * kk, idesc, (cc | tap | kk) != 0);
            umma_commit(&empty[s]);
            if (tap == 8) {
              if (kHalo) umma_commit(&aempty[hs]);
              if (cc == p.cchunks - 1) umma_commit(&tfull[slot]);
            }
          }
          __syncwarp();
          if (++s == stages) {
            s = 0;
            phase ^= 1;
          }
        }
        if (kHalo && ++hs == 2) {
          hs = 0;
          hphase ^= 1;
        }
      }
    }
  } else {  // ------------------------------------------------- epilogue
    const int q = warp & 3;              // TMEM lane quarter: conv row y = q >> 1, x = 32 (q & 1) + lane
    const int grp = (warp - 2) >> 2;     // channel group: channels [grp * 32 CPG, (grp + 1) * 32 CPG)
    const int y = q >> 1;
    const int xg = 32 * (q & 1) + lane;  // conv column of this lane
    const int cbase = grp * 32 * CPG;
    const uint32_t t_lane = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)cbase;
    const float* bch = sbias + cbase;
    uint8_t* xrow = xbuf + (grp * 64 + xg) * kXRow;
    uint32_t* gbnd = bnd + grp * CPG * 16;
    const Seg& Y = p.seg[0];
    // pooled column of this lane (even x): j = x / 2; windows x, x+1, x+2 (x+2 only inside the map)
    const int j = xg >> 1;
    const bool owner = y == 1 && (xg & 1) == 0 && j < p.PW;
    const bool three = xg + 2 < p.OW;
    uint32_t carry[CPG][16];  // conv row 2i (bf16x2 of acc + bias), y = 1 lanes
    for (int k = 0; w.valid(); w.next(), ++k) {
      const int slot = k & 1;
      mbar_wait(&tfull[slot], (uint32_t)((k >> 1) & 1));
      tc_fence_after();
      const uint32_t ts = t_lane + (uint32_t)(slot * 256);
      if (w.open) {  // tile rows (2i-1, 2i): keep row 2i
        if (y == 1) {
#pragma unroll
          for (int h = 0; h < 2 * CPG; ++h) {
            uint32_t v[16];
            tmem_ld_32x32b_x16(ts + (uint32_t)(h * 16), v);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 8; ++e)
              carry[h >> 1][(h & 1) * 8 + e] = pack_bf16x2(__uint_as_float(v[2 * e]) + bch[h * 16 + 2 * e],
                                                           __uint_as_float(v[2 * e + 1]) + bch[h * 16 + 2 * e + 1]);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[slot]);
        continue;
      }
      const bool two = w.second_row();
      if (y == 0) {  // row 2i+1 -> the exchange row of pixel xg
#pragma unroll
        for (int c = 0; c < CPG; ++c) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(ts + (uint32_t)(c * 32), v);
          tmem_wait_ld();
          uint32_t pk[16];
#pragma unroll
          for (int e = 0; e < 16; ++e)
            pk[e] = pack_bf16x2(__uint_as_float(v[2 * e]) + bch[c * 32 + 2 * e],
                                __uint_as_float(v[2 * e + 1]) + bch[c * 32 + 2 * e + 1]);
#pragma unroll
          for (int g = 0; g < 4; ++g)
            *reinterpret_cast<uint4*>(xrow + c * 64 + g * 16) = make_uint4(pk[4 * g], pk[4 * g + 1], pk[4 * g + 2], pk[4 * g + 3]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[slot]);
        named_bar_sync(1 + grp, 128);  // exchange rows written
#pragma unroll
        for (int c = 0; c < CPG; ++c)
          named_bar_sync(3 + grp, 128);  // ... and read, one channel chunk at a time (before the next tile rewrites them)
        continue;
      }
      // y == 1: rows 2i (carry), 2i+1 (exchange), 2i+2 (TMEM, when inside the map),
      // one 32-channel chunk at a time: only that chunk's maxima are live (all
      // CPG chunks at once kept 16 * CPG more registers and spilled the carry)
      named_bar_sync(1 + grp, 128);  // the exchange rows are written
      __nv_bfloat16* yp = reinterpret_cast<__nv_bfloat16*>(Y.ptr) +
                          (((long long)w.img * p.PH + w.i) * p.PW + j) * Y.ldd + Y.col0 + cbase;
#pragma unroll
      for (int c = 0; c < CPG; ++c) {
        uint32_t m[16];
        if (two) {
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {  // 16-column halves keep the live registers down
            const int h = 2 * c + hh;
            uint32_t v[16];
            tmem_ld_32x32b_x16(ts + (uint32_t)(h * 16), v);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 8; ++e)
              m[hh * 8 + e] = pack_bf16x2(__uint_as_float(v[2 * e]) + bch[h * 16 + 2 * e],
                                          __uint_as_float(v[2 * e + 1]) + bch[h * 16 + 2 * e + 1]);
          }
        }
        if (c == CPG - 1) {  // every TMEM read of this slot is done
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[slot]);
        }
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const uint4 r1 = *reinterpret_cast<const uint4*>(xrow + c * 64 + g * 16);
          const uint32_t r1w[4] = {r1.x, r1.y, r1.z, r1.w};
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int e = 4 * g + t;
            const uint32_t vm = bmax2(carry[c][e], r1w[t]);
            if (two) {
              const uint32_t r2 = m[e];
              m[e] = bmax2(vm, r2);
              carry[c][e] = r2;
            } else {
              m[e] = vm;
            }
          }
        }
        // the window of pooled column 15 (x = 30, 31, 32) crosses into the x >= 32 warp
        if (q == 3 && lane == 0) {
#pragma unroll
          for (int e = 0; e < 16; ++e) gbnd[c * 16 + e] = m[e];
        }
        named_bar_sync(3 + grp, 128);
        uint32_t o[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const uint32_t m1 = __shfl_down_sync(0xffffffffu, m[e], 1);
          uint32_t m2 = __shfl_down_sync(0xffffffffu, m[e], 2);
          if (q == 2 && lane == 30) m2 = gbnd[c * 16 + e];
          uint32_t h = bmax2(m[e], m1);
          if (three) h = bmax2(h, m2);
          o[e] = bmax2(h, 0u);  // ReLU
        }
        if (owner) {
#pragma unroll
          for (int g = 0; g < 4; ++g)
            *reinterpret_cast<uint4*>(yp + c * 32 + 8 * g) = make_uint4(o[4 * g], o[4 * g + 1], o[4 * g + 2], o[4 * g + 3]);
        }
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

template <int CPG>
int smem_fixed_bytes() {
  return 1024 + 2 * 64 * (CPG * 64 + 16) + 2 * CPG * 16 * 4 + 16 * 8 + 16 + 64 * CPG * 4;
}

}  // namespace

int launch_conv_pool(const GemmPlan* P, cudaStream_t stream) {
  const GemmParams& p = P->p;
  static bool attr = false;
  void (*const kerns[2][3])(CUtensorMap, CUtensorMap, GemmParams) = {
      {conv_pool_kernel<2, false>, conv_pool_kernel<3, false>, conv_pool_kernel<4, false>},
      {conv_pool_kernel<2, true>, conv_pool_kernel<3, true>, conv_pool_kernel<4, true>}};
  if (!attr) {
    for (auto& row : kerns)
      for (auto k : row) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  const int c = p.N / 64 - 2;
  if (c < 0 || c > 2 || p.N % 64) return set_error(MS_ERR_INVALID, "conv+pool: N must be 128, 192 or 256");
  launch_k(kerns[p.halo_slot > 0 ? 1 : 0][c], dim3(P->grid_x), dim3(kCPThreads), P->smem_bytes, stream, 1, P->tmA,
           P->tmB, p);
  return check_launch("conv_pool_kernel");
}

}  // namespace mosel

using namespace mosel;

extern "C" int ms_gemm_plan_conv_pool(void* plan, const void* X, int n_img, int H, int W_in, int C, long long c_stride,
                                      const void* Wt, int Cout, const float* bias, void* Y, long long ldy, int y_col0) {
  if (plan == nullptr || X == nullptr || Wt == nullptr || Y == nullptr) return set_error(MS_ERR_INVALID, "null pointer");
  if (Cout != 128 && Cout != 192 && Cout != 256) return set_error(MS_ERR_INVALID, "conv+pool: Cout must be 128, 192 or 256");
  const bool halo = ((W_in + 2) + 7) / 8 * 8 == kCPPitch;  // 55..62: halo rows of 64 pixels
  if ((!halo && W_in != kCPPitch) || H < 3 || n_img < 1)
    return set_error(MS_ERR_INVALID, "conv+pool: input width must be 55..62 (halo) or 64 (tap boxes), H >= 3");
  if (C < 64 || (c_stride * 2) % 16 != 0) return set_error(MS_ERR_INVALID, "conv+pool: >= 64 channels, 16-B pixel stride");
  if ((reinterpret_cast<uintptr_t>(Y) & 15) != 0 || ldy % 8 != 0 || y_col0 % 8 != 0)
    return set_error(MS_ERR_INVALID, "conv+pool: output rows must be 16-B aligned");
  GemmPlan* P = reinterpret_cast<GemmPlan*>(plan);
  memset(P, 0, sizeof(GemmPlan));
  GemmParams& p = P->p;
  p.mode = MODE_CONV_POOL;
  p.N = Cout;
  p.BN = Cout;
  p.bias = bias;
  p.relu = MS_ACT_RELU;
  p.n_img = n_img;
  p.OH = H;
  p.OW = W_in;
  p.stride = 1;
  p.pad = 1;
  p.KW = 3;
  p.M = n_img * H * W_in;
  p.cchunks = (C + kBK - 1) / kBK;
  p.PH = (H - 3 + 1) / 2 + 1;  // ceil-mode 3x3/2 pool without padding
  p.PW = (W_in - 3 + 1) / 2 + 1;
  p.units = n_img * p.PH;
  p.nseg = 1;
  p.seg[0] = Seg{0, Cout, Y, ldy, y_col0, 0};
  cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W_in, (cuuint64_t)H, (cuuint64_t)n_img};
  cuuint64_t strides[3] = {(cuuint64_t)c_stride * 2, (cuuint64_t)c_stride * 2 * W_in, (cuuint64_t)c_stride * 2 * W_in * H};
  cuuint32_t box[4] = {(cuuint32_t)kBK, (cuuint32_t)kCPPitch, (cuuint32_t)(halo ? kCPHaloRows : 2), 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  int rc = encode_bf16_map(&P->tmA, 4, X, dims, strides, box, es, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  const long long K = 9LL * p.cchunks * kBK;
  cuuint64_t wd[2] = {(cuuint64_t)K, (cuuint64_t)Cout};
  cuuint64_t ws[1] = {(cuuint64_t)K * 2};
  cuuint32_t wb[2] = {(cuuint32_t)kBK, (cuuint32_t)Cout};
  cuuint32_t we[2] = {1, 1};
  rc = encode_bf16_map(&P->tmB, 2, Wt, wd, ws, wb, we, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  P->w_ptr = Wt;
  P->w_kpad = K;
  P->w_rows = Cout;
  p.a_bytes = kBK * kCPPitch * (halo ? kCPHaloRows : 2) * 2;
  // + 2 rows of slack: the last tap's view of the last M rows reads past the halo (wrapped, unused pixels)
  p.halo_slot = halo ? ((p.a_bytes + 2 * 128) + 1023) / 1024 * 1024 : 0;  // 0: tap-box A ring
  p.b_bytes = Cout * kBK * 2;
  const int cpg = Cout / 64;
  const int fixed = cpg == 2 ? smem_fixed_bytes<2>() : cpg == 3 ? smem_fixed_bytes<3>() : smem_fixed_bytes<4>();
  int stages = (226 * 1024 - fixed - 2 * p.halo_slot) / (p.b_bytes + (halo ? 0 : kABytes));
  if (stages > 9) stages = 9;
  if (stages < 2) return set_error(MS_ERR_INVALID, "conv+pool: weight stages do not fit in shared memory");
  p.stages = stages;
  p.num_kb = 9 * p.cchunks;
  p.ksplit = 1;
  P->smem_bytes = fixed + 2 * p.halo_slot + stages * (p.b_bytes + (halo ? 0 : kABytes)) + stages * 16;
  if (P->smem_bytes > 227 * 1024) return set_error(MS_ERR_INVALID, "conv+pool plan exceeds 227 KB shared memory");
  const int sms = sm_count();
  P->grid_x = p.units < sms ? p.units : sms;
  P->grid_y = 1;
  P->tmem_cols = 512;
  return MS_OK;
}
