// Selection half of the hot path on the device:
//   * ms_policy_select — the per-job policy step, one warp per
//     job, bit-exact with apply_policy(OPTIMIZED) on a one-job scope
//     (reference scheduler.py:382-425).
//   * ms_compact_index / ms_gather_rows — request compaction: per-request
//     modality masks -> per-modality stable index lists (warp ballot + popc
//     prefix sums), inverse maps, a stable counting sort by combo
//     (strategy.py:54-60 canonical order), and vectorised row gathers into
//     contiguous modality-grouped sub-batches.
#include <cstdint>

#include <type_traits>

#include "mosel_b200.h"
#include "ptx.cuh"
#include "runtime.h"

namespace mosel {

constexpr unsigned kFull = 0xffffffffu;

// est = round-half-even(lat * factor) exactly as Python's round(int * float):
// the product is one IEEE fp64 multiply (no FMA contraction possible here).
__device__ __forceinline__ long long estimate_us(long long lat, double factor) {
  return __double2ll_rn(__dmul_rn((double)lat, factor));
}

__global__ void policy_select_kernel(const int64_t* __restrict__ lat_us, const int32_t* __restrict__ n_cand, int C,
                                     const int64_t* __restrict__ deadline_us, long long dispatch_us, double factor,
                                     int N, int32_t* __restrict__ choice) {
  const int job = (int)((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (job >= N) return;  // warp-uniform
  const int n = n_cand[job];
  const long long budget = (long long)deadline_us[job] - dispatch_us;
  const int64_t* row = lat_us + (long long)job * C;
  int best = -1;
  long long est0 = 0, est_top = 0;
  for (int base = 0; base < n; base += 32) {
    const int i = base + lane;
    const bool valid = i < n;
    const long long e = valid ? estimate_us(row[i], factor) : 0;
    const unsigned fit = __ballot_sync(kFull, valid && e <= budget);
    if (fit) best = base + 31 - __clz(fit);
    if (base == 0) est0 = __shfl_sync(kFull, e, 0);
    if (n - 1 - base < 32) est_top = __shfl_sync(kFull, e, (n - 1 - base) & 31);
  }
  if (lane != 0) return;
  int out;
  if (n <= 0) {
    out = MS_DROP;
  } else if (est_top <= budget) {
    out = n - 1;  // no violation: stays at the highest-accuracy candidate
  } else if (budget <= 0) {
    out = MS_DROP;  // compute_budget: unsavable
  } else if ((est0 + 999) / 1000 > budget / 1000) {
    out = MS_DROP;  // knapsack 1 ms grid: fastest rounds up past floor(B)
  } else {
    out = best;  // optimum then try_upgrade: largest est <= B
  }
  choice[job] = out;
}

// ---------------------------------------------------------------- compaction
constexpr int kCompactThreads = 1024;
constexpr int kMaxK = 8;

__global__ void __launch_bounds__(kCompactThreads)
    compact_index_kernel(const uint16_t* __restrict__ mask, int N, int K, int32_t* __restrict__ idx,
                         int32_t* __restrict__ inv, int32_t* __restrict__ counts, int32_t* __restrict__ offsets,
                         int32_t* __restrict__ perm) {
  __shared__ int s_excl[kMaxK][32];
  __shared__ int s_tot[kMaxK];
  __shared__ int s_base[kMaxK];
  __shared__ int s_hist[1 << kMaxK];
  __shared__ int s_cursor[1 << kMaxK];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int bins = 1 << K;
  const unsigned lt = (1u << lane) - 1u;

  if (t < K) s_base[t] = 0;
  for (int b = t; b < bins; b += kCompactThreads) s_hist[b] = 0;
  __syncthreads();

  // ---- per-modality stable index lists + combo histogram
  for (int c0 = 0; c0 < N; c0 += kCompactThreads) {
    const int i = c0 + t;
    const int m = (i < N) ? (int)mask[i] : 0;
    if (i < N) atomicAdd(&s_hist[m & (bins - 1)], 1);
    unsigned bal[kMaxK];
    for (int k = 0; k < K; ++k) {
      bal[k] = __ballot_sync(kFull, i < N && ((m >> k) & 1));
      if (lane == 0) s_excl[k][warp] = __popc(bal[k]);
    }
    __syncthreads();
    if (warp < K) {  // warp k scans the 32 warp totals of modality k
      const int k = warp;
      const int v = s_excl[k][lane];
      int incl = v;
      for (int d = 1; d < 32; d <<= 1) {
        const int y = __shfl_up_sync(kFull, incl, d);
        if (lane >= d) incl += y;
      }
      s_excl[k][lane] = incl - v;
      if (lane == 31) s_tot[k] = incl;
    }
    __syncthreads();
    if (i < N) {
      for (int k = 0; k < K; ++k) {
        if ((m >> k) & 1) {
          const int pos = s_base[k] + s_excl[k][warp] + __popc(bal[k] & lt);
          idx[(long long)k * N + pos] = i;
          inv[(long long)k * N + i] = pos;
        } else {
          inv[(long long)k * N + i] = -1;
        }
      }
    }
    __syncthreads();
    if (t < K) s_base[t] += s_tot[t];
    __syncthreads();
  }
  if (t < K) counts[t] = s_base[t];

  // ---- exclusive scan of the combo histogram -> offsets (bins <= 256)
  if (t == 0) {
    int acc = 0;
    for (int b = 0; b < bins; ++b) {
      offsets[b] = acc;
      s_cursor[b] = acc;
      acc += s_hist[b];
    }
    offsets[bins] = acc;
  }
  __syncthreads();

  // ---- stable placement by mask (match_any ranks within the warp)
  for (int c0 = 0; c0 < N; c0 += kCompactThreads) {
    const int i = c0 + t;
    const int m = (i < N) ? (int)mask[i] & (bins - 1) : bins;  // sentinel bin for tail lanes
    const unsigned peers = __match_any_sync(kFull, m);
    const int rank = __popc(peers & lt);
    const int leader = __ffs(peers) - 1;
    // serialise warps in order so earlier warps claim earlier slots
    for (int w = 0; w < kCompactThreads / 32; ++w) {
      if (warp == w && i < N) {
        int slot_base = 0;
        if (lane == leader) slot_base = atomicAdd(&s_cursor[m], __popc(peers));
        slot_base = __shfl_sync(peers, slot_base, leader);
        perm[slot_base + rank] = i;
      }
      __syncthreads();
    }
  }
}

// dst[j] = src[slot ? slot[idx[j]] : idx[j]], j < *count; blockIdx.y = row
__global__ void gather_rows_kernel(const uint4* __restrict__ src, long long row_vecs, const int32_t* __restrict__ slot,
                                   const int32_t* __restrict__ idx, const int32_t* __restrict__ count,
                                   uint4* __restrict__ dst) {
  const int n = *count;
  for (int j = blockIdx.y; j < n; j += gridDim.y) {
    int r = idx[j];
    if (slot) r = slot[r];
    const uint4* s = src + (long long)r * row_vecs;
    uint4* d = dst + (long long)j * row_vecs;
    const long long step = (long long)gridDim.x * blockDim.x;
    long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    for (; v + 3 * step < row_vecs; v += 4 * step) {
      const uint4 a = __ldcs(s + v), b = __ldcs(s + v + step), c = __ldcs(s + v + 2 * step),
                  e = __ldcs(s + v + 3 * step);
      d[v] = a;
      d[v + step] = b;
      d[v + 2 * step] = c;
      d[v + 3 * step] = e;
    }
    for (; v < row_vecs; v += step) d[v] = __ldcs(s + v);
  }
}

// Padding gather: a source row is `lines` lines of `width` pixels with c_src
// channels; the destination row has c_dst (multiple of 8, >= c_src) channels
// and `pad_w` zero pixels on both ends of every line (the first conv's
// window padding, so its TMA windows never leave the line).  One thread =
// one destination pixel x 8 channels (one 16-B store).
// One CTA = one source line of one request at a time: the line (width *
// c_src elements, 16-B aligned) is staged into shared memory with 16-B vector
// loads, then each thread emits whole destination pixels (c_dst/8 16-B
// stores, zero pad channels / pad pixels), converting uint8 on the fly.
constexpr int kMaxLineBytes = 16384;
// V = channels per vector store: 8 (uint4, c_dst % 8 == 0) or 4 (uint2, c_dst == 4).
// frame_h > 0: the source lines are frames of frame_h rows and every frame
// gets pad_h zero rows above and below in the destination (rows the kernel
// never writes: the destination buffer is zeroed once at allocation).
template <bool U8, int V>
__global__ void __launch_bounds__(256) gather_rows_pad_kernel(const void* __restrict__ src_v, long long lines,
                                                              int width, int c_src, int c_dst, int pad_w,
                                                              float u8_scale, float u8_bias,
                                                              const int32_t* __restrict__ slot,
                                                              const int32_t* __restrict__ idx,
                                                              const int32_t* __restrict__ count,
                                                              void* __restrict__ dst_v, int frame_h, int pad_h,
                                                              long long plane_vecs, int per_cap, int pdl_mode) {
  // PDL chain across one pass's gathers (ms_compact, pdl_mode 1 then 2): the first waits for the
  // index kernel, then lets the next gather start; later gathers start at
  // once and wait for their predecessor only before exiting, so gathers of
  // different modalities overlap and the last one's completion still implies
  // all of them (what a PDL successor's griddepcontrol.wait observes)
  if (pdl_mode != 2) pdl_wait();  // 0: standalone launch, 1: first of a chain
  pdl_trigger();
  typedef typename std::conditional<V == 8, uint4, uint2>::type vec_t;
  __shared__ __align__(16) unsigned char line_buf[kMaxLineBytes];
  __shared__ long long s_dline[32];
  vec_t* dst = reinterpret_cast<vec_t*>(dst_v);
  const int n = *count;
  const int esz = U8 ? 1 : 2;
  const int line_bytes = width * c_src * esz;
  const int gv = c_dst / V;
  const int wd = width + 2 * pad_w;
  const long long dst_lines = frame_h > 0 ? lines + (lines / frame_h) * 2LL * pad_h : lines;
  for (int j = blockIdx.y; j < n; j += gridDim.y) {
    int r = idx[j];
    if (slot) r = slot[r];
    const unsigned char* srow = reinterpret_cast<const unsigned char*>(src_v) + (long long)r * lines * line_bytes;
    vec_t* drow = dst + (long long)j * dst_lines * wd * gv;
    const int per = min(per_cap, max(1, kMaxLineBytes / line_bytes));  // lines staged per round
    for (long long ln0 = (long long)blockIdx.x * per; ln0 < lines; ln0 += (long long)gridDim.x * per) {
      const int nl = (int)min((long long)per, lines - ln0);
      __syncthreads();
      const uint4* s4 = reinterpret_cast<const uint4*>(srow + ln0 * line_bytes);
      for (int i = threadIdx.x; i < nl * line_bytes / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(line_buf)[i] = __ldcs(s4 + i);
      if (threadIdx.x < nl) {  // destination line of each staged line (frame row padding)
        const long long ln = ln0 + threadIdx.x;
        s_dline[threadIdx.x] = frame_h > 0 ? (ln / frame_h) * (frame_h + 2LL * pad_h) + pad_h + ln % frame_h : ln;
      }
      __syncthreads();
      if constexpr (V == 4) {
        if ((wd & 1) == 0 && gv == 3) {  // 12-channel pixels: two per thread, three 16-B stores
          const int wq = wd >> 1;
          int li = threadIdx.x / wq, pq = threadIdx.x - li * wq;
          const int step_l = blockDim.x / wq, step_p = blockDim.x - step_l * wq;
          for (; li < nl; li += step_l, pq += step_p) {
            if (pq >= wq) {
              pq -= wq;
              ++li;
              if (li >= nl) break;
            }
            const unsigned char* lb = line_buf + li * line_bytes;
            unsigned short v[24];
#pragma unroll
            for (int i = 0; i < 24; ++i) v[i] = 0;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int x = 2 * pq + h - pad_w;
              if (x >= 0 && x < width) {
#pragma unroll
                for (int c = 0; c < 12; ++c) {
                  if (c < c_src) {
                    if (U8) {
                      const __nv_bfloat16 b =
                          __float2bfloat16_rn(fmaf((float)lb[x * c_src + c], u8_scale, u8_bias));
                      v[12 * h + c] = *reinterpret_cast<const unsigned short*>(&b);
                    } else {
                      v[12 * h + c] = reinterpret_cast<const unsigned short*>(lb)[x * c_src + c];
                    }
                  }
                }
              }
            }
            if (plane_vecs > 0) {  // planar: channels 4q..4q+3 of both pixels -> plane q
              const long long pix = ((long long)j * dst_lines + s_dline[li]) * wd + 2 * pq;
#pragma unroll
              for (int q = 0; q < 3; ++q)
                *reinterpret_cast<uint4*>(dst + q * plane_vecs + pix) =
                    make_uint4(v[4 * q] | ((unsigned)v[4 * q + 1] << 16), v[4 * q + 2] | ((unsigned)v[4 * q + 3] << 16),
                               v[12 + 4 * q] | ((unsigned)v[12 + 4 * q + 1] << 16),
                               v[12 + 4 * q + 2] | ((unsigned)v[12 + 4 * q + 3] << 16));
              continue;
            }
            uint4* d4 = reinterpret_cast<uint4*>(drow + (s_dline[li] * wd + 2 * pq) * 3);
#pragma unroll
            for (int q = 0; q < 3; ++q)
              d4[q] = make_uint4(v[8 * q] | ((unsigned)v[8 * q + 1] << 16), v[8 * q + 2] | ((unsigned)v[8 * q + 3] << 16),
                                 v[8 * q + 4] | ((unsigned)v[8 * q + 5] << 16),
                                 v[8 * q + 6] | ((unsigned)v[8 * q + 7] << 16));
          }
          continue;
        }
        if ((wd & 1) == 0 && gv == 1) {  // 4-channel pixels: two per thread, one 16-B store
          const int wq = wd >> 1;
          int li = threadIdx.x / wq, pq = threadIdx.x - li * wq;
          const int step_l = blockDim.x / wq, step_p = blockDim.x - step_l * wq;
          for (; li < nl; li += step_l, pq += step_p) {
            if (pq >= wq) {
              pq -= wq;
              ++li;
              if (li >= nl) break;
            }
            const unsigned char* lb = line_buf + li * line_bytes;
            unsigned short v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int x = 2 * pq + h - pad_w;
              if (x >= 0 && x < width) {
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                  if (c < c_src) {
                    if (U8) {
                      const __nv_bfloat16 b =
                          __float2bfloat16_rn(fmaf((float)lb[x * c_src + c], u8_scale, u8_bias));
                      v[4 * h + c] = *reinterpret_cast<const unsigned short*>(&b);
                    } else {
                      v[4 * h + c] = reinterpret_cast<const unsigned short*>(lb)[x * c_src + c];
                    }
                  }
                }
              }
            }
            *reinterpret_cast<uint4*>(drow + (s_dline[li] * wd + 2 * pq)) =
                make_uint4(v[0] | ((unsigned)v[1] << 16), v[2] | ((unsigned)v[3] << 16),
                           v[4] | ((unsigned)v[5] << 16), v[6] | ((unsigned)v[7] << 16));
          }
          continue;
        }
      }
      int li = threadIdx.x / wd, px = threadIdx.x - li * wd;  // (line, pixel), advanced without divisions
      const int step_l = blockDim.x / wd, step_p = blockDim.x - step_l * wd;
      for (; li < nl; li += step_l, px += step_p) {
        if (px >= wd) {
          px -= wd;
          ++li;
          if (li >= nl) break;
        }
        vec_t* d = drow + (s_dline[li] * wd + px) * gv;
        const int x = px - pad_w;
        const unsigned char* lb = line_buf + li * line_bytes;
        for (int g = 0; g < gv; ++g) {
          unsigned short v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
          if (x >= 0 && x < width) {
#pragma unroll
            for (int i = 0; i < V; ++i) {
              const int c = g * V + i;
              if (c < c_src) {
                if (U8) {
                  const __nv_bfloat16 b = __float2bfloat16_rn(fmaf((float)lb[x * c_src + c], u8_scale, u8_bias));
                  v[i] = *reinterpret_cast<const unsigned short*>(&b);
                } else {
                  v[i] = reinterpret_cast<const unsigned short*>(lb)[x * c_src + c];
                }
              }
            }
          }
          if constexpr (V == 8)
            d[g] = make_uint4(v[0] | ((unsigned)v[1] << 16), v[2] | ((unsigned)v[3] << 16),
                              v[4] | ((unsigned)v[5] << 16), v[6] | ((unsigned)v[7] << 16));
          else
            d[g] = make_uint2(v[0] | ((unsigned)v[1] << 16), v[2] | ((unsigned)v[3] << 16));
        }
      }
    }
  }
  if (pdl_mode == 2) pdl_wait();
}

// generic fallback (line not 16-B aligned or too long): one thread = one
// destination pixel x 8 channels, scalar loads
template <bool U8>
__global__ void gather_rows_pad_scalar_kernel(const void* __restrict__ src_v, long long lines, int width, int c_src,
                                              int c_dst, int pad_w, float u8_scale, float u8_bias,
                                              const int32_t* __restrict__ slot, const int32_t* __restrict__ idx,
                                              const int32_t* __restrict__ count, uint4* __restrict__ dst) {
  const int n = *count;
  const int g8 = c_dst / 8;
  const int wd = width + 2 * pad_w;
  const long long work = lines * wd * g8;
  const long long src_row = lines * width * c_src;
  for (int j = blockIdx.y; j < n; j += gridDim.y) {
    int r = idx[j];
    if (slot) r = slot[r];
    uint4* d = dst + (long long)j * work;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < work;
         t += (long long)gridDim.x * blockDim.x) {
      const long long px = t / g8;
      const int c0 = (int)(t - px * g8) * 8;
      const long long line = px / wd;
      const int x = (int)(px - line * wd) - pad_w;
      unsigned short v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      if (x >= 0 && x < width) {
        const long long off = (long long)r * src_row + (line * width + x) * c_src + c0;
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (c0 + i < c_src) {
            if (U8) {
              const __nv_bfloat16 b = __float2bfloat16_rn(
                  fmaf((float)reinterpret_cast<const unsigned char*>(src_v)[off + i], u8_scale, u8_bias));
              v[i] = *reinterpret_cast<const unsigned short*>(&b);
            } else {
              v[i] = reinterpret_cast<const unsigned short*>(src_v)[off + i];
            }
          }
      }
      d[t] = make_uint4(v[0] | ((unsigned)v[1] << 16), v[2] | ((unsigned)v[3] << 16),
                        v[4] | ((unsigned)v[5] << 16), v[6] | ((unsigned)v[7] << 16));
    }
  }
}

static int gather_pad_launch(const void* src, long long lines, int width, int c_src, int c_dst, int pad_w,
                             const int32_t* slot, const int32_t* idx, const int32_t* count, int max_rows, void* dst,
                             cudaStream_t st, int src_u8 = 0, float u8_scale = 1.0f, float u8_bias = 0.0f,
                             int frame_h = 0, int pad_h = 0, long long plane_stride = 0, int pdl_mode = 0) {
  if (c_dst % 4 != 0 || c_src > c_dst || c_src < 1 || pad_w < 0 || width < 1)
    return set_error(MS_ERR_INVALID, "gather: need 1 <= c_src <= c_dst, c_dst % 4 == 0, pad_w >= 0");
  if (frame_h < 0 || pad_h < 0 || (frame_h > 0 && lines % frame_h != 0))
    return set_error(MS_ERR_INVALID, "gather: frame_h must divide lines, pad_h >= 0");
  if (max_rows <= 0) return MS_OK;
  const int gy = max_rows < 65535 ? max_rows : 65535;
  const long long line_bytes = (long long)width * c_src * (src_u8 ? 1 : 2);
  if (plane_stride > 0 && (c_dst != 12 || ((width + 2 * pad_w) & 1) != 0 || line_bytes % 16 != 0 ||
                           line_bytes > kMaxLineBytes || plane_stride % 4 != 0))
    return set_error(MS_ERR_INVALID, "gather: planar output needs 12 destination channels, even padded width");
  if (line_bytes % 16 == 0 && line_bytes <= kMaxLineBytes) {
    static const int per_env = getenv("MS_GATHER_LINES") ? atoi(getenv("MS_GATHER_LINES")) : 0;  // A/B
    const int per_cap = per_env > 0 ? per_env : 32;
    const long long per = line_bytes > 0 ? (kMaxLineBytes / line_bytes < per_cap ? kMaxLineBytes / line_bytes : per_cap) : 1;
    long long bx = (lines + per - 1) / per;
    if (bx > 64) bx = 64;
    if (bx < 1) bx = 1;
    const dim3 grid((unsigned)bx, (unsigned)gy);
    const float sc = src_u8 ? u8_scale : 1.0f, bi = src_u8 ? u8_bias : 0.0f;
    if (c_dst % 8 != 0) {  // 8-byte vector stores (4-channel groups)
      if (src_u8)
        launch_k(gather_rows_pad_kernel<true, 4>, grid, dim3(256), 0, st, 1, src, lines, width, c_src, c_dst, pad_w, sc, bi, slot,
                                                              idx, count, dst, frame_h, pad_h, plane_stride / 4, per_cap, pdl_mode);
      else
        launch_k(gather_rows_pad_kernel<false, 4>, grid, dim3(256), 0, st, 1, src, lines, width, c_src, c_dst, pad_w, sc, bi, slot,
                                                               idx, count, dst, frame_h, pad_h, plane_stride / 4, per_cap, pdl_mode);
    } else if (src_u8) {
      launch_k(gather_rows_pad_kernel<true, 8>, grid, dim3(256), 0, st, 1, src, lines, width, c_src, c_dst, pad_w, sc, bi, slot,
                                                            idx, count, dst, frame_h, pad_h, plane_stride / 4, per_cap, pdl_mode);
    } else {
      launch_k(gather_rows_pad_kernel<false, 8>, grid, dim3(256), 0, st, 1, src, lines, width, c_src, c_dst, pad_w, sc, bi, slot,
                                                             idx, count, dst, frame_h, pad_h, plane_stride / 4, per_cap, pdl_mode);
    }
  } else {
    if (c_dst % 8 != 0 || frame_h > 0)
      return set_error(MS_ERR_INVALID, "gather: 4-channel / frame-padded rows need 16-B aligned source lines");
    const long long work = lines * (width + 2LL * pad_w) * (c_dst / 8);
    long long bx = (work + 255) / 256;
    if (bx > 1024) bx = 1024;
    if (bx < 1) bx = 1;
    if (src_u8)
      gather_rows_pad_scalar_kernel<true><<<dim3((unsigned)bx, (unsigned)gy), 256, 0, st>>>(
          src, lines, width, c_src, c_dst, pad_w, u8_scale, u8_bias, slot, idx, count, reinterpret_cast<uint4*>(dst));
    else
      gather_rows_pad_scalar_kernel<false><<<dim3((unsigned)bx, (unsigned)gy), 256, 0, st>>>(
          src, lines, width, c_src, c_dst, pad_w, 1.0f, 0.0f, slot, idx, count, reinterpret_cast<uint4*>(dst));
  }
  return check_launch("gather_rows_pad_kernel");
}

static int gather_launch(const void* src, long long row_bytes, const int32_t* slot, const int32_t* idx,
                         const int32_t* count, int max_rows, void* dst, cudaStream_t st) {
  if (row_bytes % 16 != 0) return set_error(MS_ERR_INVALID, "row_bytes must be a multiple of 16");
  if (max_rows <= 0) return MS_OK;
  const long long vecs = row_bytes / 16;
  long long bx = (vecs + 256 * 4 - 1) / (256 * 4);
  if (bx > 512) bx = 512;
  if (bx < 1) bx = 1;
  int gy = max_rows < 65535 ? max_rows : 65535;
  dim3 grid((unsigned)bx, (unsigned)gy);
  gather_rows_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const uint4*>(src), vecs, slot, idx, count,
                                           reinterpret_cast<uint4*>(dst));
  return check_launch("gather_rows_kernel");
}

}  // namespace mosel

using namespace mosel;

extern "C" {

int ms_policy_select(const int64_t* lat_us, const int32_t* credit, const int32_t* n_cand, int C,
                     const int64_t* deadline_us, int64_t dispatch_us, double factor, int N, int32_t* choice,
                     void* stream) {
  (void)credit;  // frontier credits are strictly increasing: the argmax is the largest feasible index
  if (N < 0 || C < 1) return set_error(MS_ERR_INVALID, "policy_select: bad shape");
  if (N == 0) return MS_OK;
  if (!lat_us || !n_cand || !deadline_us || !choice) return set_error(MS_ERR_INVALID, "policy_select: null pointer");
  if (!(factor > 0.0)) return set_error(MS_ERR_INVALID, "policy_select: factor must be positive");
  const int threads = 256;
  const long long warps = N;
  const int blocks = (int)((warps * 32 + threads - 1) / threads);
  policy_select_kernel<<<blocks, threads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      lat_us, n_cand, C, deadline_us, (long long)dispatch_us, factor, N, choice);
  return check_launch("policy_select_kernel");
}

int ms_compact_index(const uint16_t* mask, int N, int K, int32_t* idx, int32_t* inv, int32_t* counts,
                     int32_t* combo_offsets, int32_t* perm, void* stream) {
  if (K < 1 || K > kMaxK) return set_error(MS_ERR_INVALID, "compact: K must be in 1..8");
  if (N < 0) return set_error(MS_ERR_INVALID, "compact: N must be >= 0");
  if (!mask && N > 0) return set_error(MS_ERR_INVALID, "compact: null mask");
  compact_index_kernel<<<1, kCompactThreads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(mask, N, K, idx, inv,
                                                                                         counts, combo_offsets, perm);
  return check_launch("compact_index_kernel");
}

int ms_gather_rows(const void* src, long long row_bytes, const int32_t* slot, const int32_t* idx,
                   const int32_t* count, int max_rows, void* dst, void* stream) {
  if (!src || !idx || !count || !dst) return set_error(MS_ERR_INVALID, "gather_rows: null pointer");
  return gather_launch(src, row_bytes, slot, idx, count, max_rows, dst, reinterpret_cast<cudaStream_t>(stream));
}

int ms_gather_rows_pad(const void* src, long long lines, int width, int c_src, int c_dst, int pad_w,
                       const int32_t* slot, const int32_t* idx, const int32_t* count, int max_rows, void* dst,
                       void* stream) {
  if (!src || !idx || !count || !dst) return set_error(MS_ERR_INVALID, "gather_rows_pad: null pointer");
  return gather_pad_launch(src, lines, width, c_src, c_dst, pad_w, slot, idx, count, max_rows, dst,
                           reinterpret_cast<cudaStream_t>(stream));
}

int ms_compact(const uint16_t* mask, int N, int K, const void* const* X, const MsRowDesc* rows,
               const int32_t* slot, void* const* G, int32_t* idx, int32_t* inv, int32_t* counts,
               int32_t* combo_offsets, int32_t* perm, void* stream) {
  int rc = ms_compact_index(mask, N, K, idx, inv, counts, combo_offsets, perm, stream);
  if (rc) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  bool chained = false;  // the previous launch was a padded gather of this chain
  for (int k = 0; k < K; ++k) {
    if (X == nullptr || G == nullptr || rows == nullptr || X[k] == nullptr || G[k] == nullptr) continue;
    const MsRowDesc& r = rows[k];
    const long long bytes = r.lines * (long long)r.width * r.c_src * 2;
    const bool framed = r.frame_h > 0 && r.pad_h > 0;
    const int32_t* sk = slot ? slot + r.slot_off : nullptr;  // per-modality pool rows
    if (!r.src_u8 && r.c_src == r.c_dst && r.pad_w == 0 && !framed && r.plane_stride == 0 && bytes % 16 == 0) {
      rc = gather_launch(X[k], bytes, sk, idx + (long long)k * N, counts + k, N, G[k], st);
      chained = false;  // a plain launch ends the PDL chain (the next gather waits at its start again)
    } else {
      rc = gather_pad_launch(X[k], r.lines, r.width, r.c_src, r.c_dst, r.pad_w, sk, idx + (long long)k * N,
                             counts + k, N, G[k], st, r.src_u8, r.u8_scale, r.u8_bias, framed ? r.frame_h : 0,
                             framed ? r.pad_h : 0, r.plane_stride, chained ? 2 : 1);
      chained = true;
    }
    if (rc) return rc;
  }
  return MS_OK;
}

}  // extern "C"
