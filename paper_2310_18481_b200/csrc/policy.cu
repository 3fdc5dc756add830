// Coupled queue policy on the device: the reference's
// OPTIMIZED dropping policy over a whole EDF queue,
//
//   apply_policy(OPTIMIZED)          scheduler.py:382-425
//     detect_violation / budget      scheduler.py:187-233 (prefix sums of est)
//     reassign_optimized (MCKP)      scheduler.py:236-326 (grid DP + reconstruction)
//     try_upgrade                    scheduler.py:366-379
//
// in ONE single-CTA launch.  Control flow (violation search, budget, drops,
// upgrades) runs on thread 0 over shared-memory tables, the reconstruction on
// one warp (candidates in parallel, ballot); the knapsack's value/accuracy
// rows (one per job, `width` grid cells) are computed by all threads, one
// grid cell per thread, candidates in frontier order so ties resolve exactly
// as the reference's vectorised numpy update does (max credit, then max
// min-accuracy, then earliest candidate).  Estimates are round-half-even of
// latency * factor in fp64 (__double2ll_rn == Python round), grid units are
// ceil(est / grid), prefix caps use floor division -- bit-exact with the
// reference on tests/golden/queue_policy_cases.json.
//
// The try_upgrade walk is incremental: with the queue violation-free before
// every attempt (the reassign loop exits only then, and only upgrades that
// keep it so are kept), "detect_violation() is not None" after raising job
// p's estimate by delta is exactly "delta > min_{k >= p} (deadline_k -
// completion_k)", so each attempt is O(1) instead of the reference's O(n).
#include <climits>
#include <cstdint>

#include "mosel_b200.h"
#include "ptx.cuh"
#include "runtime.h"

namespace mosel {

constexpr int kPolThreads = 512;
constexpr int kPolSmemMax = 220 * 1024;  // dynamic shared memory budget (per-job tables)

__device__ __forceinline__ long long est_us(long long lat, double f) {
  return __double2ll_rn((double)lat * f);  // Python round(): half-even
}
__device__ __forceinline__ long long floordiv(long long a, long long b) {  // b > 0
  long long q = a / b;
  if ((a % b) != 0 && a < 0) --q;
  return q;
}

// Per-job tables in dynamic shared memory (bytes per job; see policy_smem_bytes).
// The factor is fixed for the launch, so every candidate's estimate and grid
// units are computed once, in parallel, and the serial control flow (thread
// 0) reads shared memory only -- the round-1 kernel read global memory there
// and spent most of its time in L2 round trips at 128 queued jobs.
struct PolSmem {
  long long* est;   // [n * C]
  long long* dl;    // [n]
  long long* caps;  // [n]
  long long* comp;  // [n]
  long long* sfx;   // [n]
  int32_t* units;   // [n * C]
  int32_t* ncand;   // [n]
  int32_t* asg;     // [n]
  int32_t* scope;   // [n]
  uint8_t* alive;   // [n]
};
__host__ __device__ inline long long policy_smem_bytes(int n, int C) {
  return (long long)n * C * (8 + 4) + (long long)n * (8 * 4 + 4 * 3 + 1) + 64;
}
__device__ inline PolSmem carve(uint8_t* base, int n, int C) {
  PolSmem t;
  uint8_t* q = base;
  t.est = reinterpret_cast<long long*>(q);
  q += (size_t)n * C * 8;
  t.dl = reinterpret_cast<long long*>(q);
  q += (size_t)n * 8;
  t.caps = reinterpret_cast<long long*>(q);
  q += (size_t)n * 8;
  t.comp = reinterpret_cast<long long*>(q);
  q += (size_t)n * 8;
  t.sfx = reinterpret_cast<long long*>(q);
  q += (size_t)n * 8;
  t.units = reinterpret_cast<int32_t*>(q);
  q += (size_t)n * C * 4;
  t.ncand = reinterpret_cast<int32_t*>(q);
  q += (size_t)n * 4;
  t.asg = reinterpret_cast<int32_t*>(q);
  q += (size_t)n * 4;
  t.scope = reinterpret_cast<int32_t*>(q);
  q += (size_t)n * 4;
  t.alive = q;
  return t;
}

__global__ void __launch_bounds__(kPolThreads) policy_apply_kernel(
    int n, int C, const long long* __restrict__ lat, const int32_t* __restrict__ credit,
    const double* __restrict__ acc, const int32_t* __restrict__ n_cand, const long long* __restrict__ deadline,
    int32_t* __restrict__ assigned_io, long long now_us, long long running_finish_us, int has_running,
    double factor, long long grid_us, long long* __restrict__ hval, double* __restrict__ hworst,
    long long hist_cells, int32_t* __restrict__ status) {
  extern __shared__ __align__(16) uint8_t pol_smem[];
  const PolSmem S = carve(pol_smem, n, C);
  __shared__ int s_m, s_width, s_v, s_phase;
  __shared__ long long s_best_val[kPolThreads / 32];
  __shared__ double s_best_w[kPolThreads / 32];
  __shared__ int s_best_t[kPolThreads / 32];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) *status = 0;
  for (int j = tid; j < n; j += blockDim.x) {
    S.asg[j] = assigned_io[j];
    S.alive[j] = 1;
    S.dl[j] = deadline[j];
    S.ncand[j] = n_cand[j];
  }
  for (int i = tid; i < n * C; i += blockDim.x) {
    const long long e = est_us(lat[i], factor);
    S.est[i] = e;
    S.units[i] = (int32_t)((e + grid_us - 1) / grid_us);  // e >= 0: -(-e // grid)
  }
  __syncthreads();
  const long long dispatch = has_running ? max(now_us, running_finish_us) : now_us;

  // ------------------------------------------------ violation / MCKP loop
  for (;;) {
    if (tid == 0) {
      // detect_violation: first queued job whose prefix completion > deadline
      long long t = dispatch;
      int v = -1;
      for (int j = 0; j < n; ++j) {
        if (!S.alive[j]) continue;
        t += S.est[j * C + S.asg[j]];
        if (t > S.dl[j]) {
          v = j;
          break;
        }
      }
      s_v = v;
      s_phase = 0;  // 0: stop, 1: drop v, 2: run the knapsack
      if (v >= 0) {
        const long long budget = S.dl[v] - dispatch;  // compute_budget (start = dispatch)
        s_phase = 1;
        if (budget > 0) {
          // scope = queued jobs up to and including v; prefix caps in grid units
          int m = 0;
          long long run = 0, min_cap = 0;
          for (int j = 0; j <= v; ++j) {
            if (!S.alive[j]) continue;
            long long mx = 0;
            for (int c = 0; c < S.ncand[j]; ++c) mx = max(mx, (long long)S.units[j * C + c]);
            run += mx;
            long long cap = budget / grid_us;
            cap = run < cap ? run : cap;
            const long long dl = floordiv(S.dl[j] - dispatch, grid_us);
            cap = dl < cap ? dl : cap;
            S.caps[m] = cap;
            min_cap = (m == 0 || cap < min_cap) ? cap : min_cap;
            S.scope[m++] = j;
          }
          if (min_cap >= 0) {
            const long long width = S.caps[m - 1] + 1;
            if (width * (long long)(m + 1) > hist_cells) {
              *status = 1;  // the caller sizes the workspace (policy_ws_cells) so this never fires
            } else {
              s_m = m;
              s_width = (int)width;
              s_phase = 2;
            }
          }
        }
      }
    }
    __syncthreads();
    if (*status != 0) return;
    if (s_phase == 0) break;
    if (s_phase == 2) {
      const int m = s_m, width = s_width;
      // row 0: val[0] = 0, else -1; worst = +inf
      for (int t = tid; t < width; t += blockDim.x) {
        hval[t] = t == 0 ? 0 : -1;
        hworst[t] = INFINITY;
      }
      __syncthreads();
      for (int i = 0; i < m; ++i) {
        const int j = S.scope[i];
        const long long* pv = hval + (long long)i * width;
        const double* pw = hworst + (long long)i * width;
        long long* nv = hval + (long long)(i + 1) * width;
        double* nw = hworst + (long long)(i + 1) * width;
        const long long top = min(S.caps[i], (long long)width - 1);
        const int nc = S.ncand[j];
        for (int t = tid; t < width; t += blockDim.x) {
          long long dv = -1;
          double dw = -INFINITY;
          if (t <= top) {
            for (int c = 0; c < nc; ++c) {
              const int d = S.units[j * C + c];
              if (d > top || t < d) continue;
              const long long sv = pv[t - d];
              if (sv < 0) continue;
              const long long cv = sv + credit[(long long)j * C + c];
              const double a = acc[(long long)j * C + c];
              const double sw = pw[t - d];
              const double cw = sw < a ? sw : a;
              if (cv > dv || (cv == dv && cw > dw)) {
                dv = cv;
                dw = cw;
              }
            }
          }
          nv[t] = dv;
          nw[t] = dw;
        }
        __syncthreads();
      }
      // best cell: max value, then max worst accuracy, then smallest t
      const long long* fv = hval + (long long)m * width;
      const double* fw = hworst + (long long)m * width;
      long long bv = -1;
      double bw = -INFINITY;
      int bt = 0x7fffffff;
      for (int t = tid; t < width; t += blockDim.x) {
        const long long v = fv[t];
        if (v < 0) continue;
        const double w = fw[t];
        if (v > bv || (v == bv && (w > bw || (w == bw && t < bt)))) {
          bv = v;
          bw = w;
          bt = t;
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const long long ov = __shfl_down_sync(0xffffffffu, bv, o);
        const double ow = __shfl_down_sync(0xffffffffu, bw, o);
        const int ot = __shfl_down_sync(0xffffffffu, bt, o);
        if (ov > bv || (ov == bv && (ow > bw || (ow == bw && ot < bt)))) {
          bv = ov;
          bw = ow;
          bt = ot;
        }
      }
      if (lane == 0) {
        s_best_val[warp] = bv;
        s_best_w[warp] = bw;
        s_best_t[warp] = bt;
      }
      __syncthreads();
      if (warp == 0) {
        // every lane reduces the per-warp bests (same order, same result)
        bv = -1;
        bw = -INFINITY;
        bt = 0x7fffffff;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
          const long long ov = s_best_val[w];
          const double ow = s_best_w[w];
          const int ot = s_best_t[w];
          if (ov > bv || (ov == bv && (ow > bw || (ow == bw && ot < bt)))) {
            bv = ov;
            bw = ow;
            bt = ot;
          }
        }
        if (bv < 0) {
          if (lane == 0) S.alive[s_v] = 0;  // no feasible assignment: drop the violator
        } else {
          // reconstruction from the back: the fastest (first) candidate that
          // reproduces the optimum at each step -- lanes test candidates in
          // parallel, the lowest matching index wins (ballot)
          long long want_v = bv;
          double want_w = bw;
          int t = bt;
          for (int i = m - 1; i >= 0; --i) {
            const int j = S.scope[i];
            const long long* pv = hval + (long long)i * width;
            const double* pw = hworst + (long long)i * width;
            const int nc = S.ncand[j];
            int pick = -1;
            for (int c0 = 0; c0 < nc && pick < 0; c0 += 32) {
              const int c = c0 + lane;
              bool ok = false;
              if (c < nc) {
                const int d = S.units[j * C + c];
                const int s = t - d;
                if (s >= 0 && t <= S.caps[i] && pv[s] >= 0) {
                  const double a = acc[(long long)j * C + c];
                  const double mw = pw[s] < a ? pw[s] : a;
                  ok = pv[s] + credit[(long long)j * C + c] == want_v && mw == want_w;
                }
              }
              const unsigned bal = __ballot_sync(0xffffffffu, ok);
              if (bal) pick = c0 + __ffs(bal) - 1;
            }
            if (pick >= 0) {
              const int s = t - S.units[j * C + pick];
              if (lane == 0) S.asg[j] = pick;
              t = s;
              want_v = pv[s];
              want_w = pw[s];
            }
          }
        }
      }
      __syncthreads();
    } else {  // phase 1: budget <= 0 or infeasible caps -> drop the violator
      if (tid == 0) S.alive[s_v] = 0;
      __syncthreads();
    }
  }

  // ----------------------------------------------------------- try_upgrade
  if (tid == 0) {
    // completion times and suffix-min slack over the queued jobs (no violation)
    long long t = dispatch;
    for (int j = 0; j < n; ++j) {
      if (!S.alive[j]) continue;
      t += S.est[j * C + S.asg[j]];
      S.comp[j] = t;
    }
    auto rebuild = [&]() {
      long long mn = LLONG_MAX;
      for (int j = n - 1; j >= 0; --j) {
        if (S.alive[j]) {
          const long long sl = S.dl[j] - S.comp[j];
          mn = sl < mn ? sl : mn;
        }
        S.sfx[j] = mn;
      }
    };
    rebuild();
    bool moved = true;
    while (moved) {
      moved = false;
      for (int j = 0; j < n; ++j) {
        if (!S.alive[j]) continue;
        while (S.asg[j] + 1 < S.ncand[j]) {
          const long long delta = S.est[j * C + S.asg[j] + 1] - S.est[j * C + S.asg[j]];
          if (delta > S.sfx[j]) break;  // would create a violation at or after j
          S.asg[j] += 1;
          moved = true;
          if (delta != 0) {
            for (int k = j; k < n; ++k)
              if (S.alive[k]) S.comp[k] += delta;
            rebuild();
          }
        }
      }
    }
  }
  __syncthreads();
  for (int j = tid; j < n; j += blockDim.x) assigned_io[j] = S.alive[j] ? S.asg[j] : -1;
}

}  // namespace mosel

using namespace mosel;

extern "C" {

int ms_policy_apply(int n, int C, const int64_t* lat_us, const int32_t* credit, const double* acc,
                    const int32_t* n_cand, const int64_t* deadline_us, int32_t* assigned, int64_t now_us,
                    int64_t running_finish_us, int has_running, double factor, int64_t grid_us, void* ws,
                    long long ws_bytes, int32_t* status, void* stream) {
  if (n < 0 || C < 1 || C > 64) return set_error(MS_ERR_INVALID, "policy_apply: bad shape");
  if (n == 0) return MS_OK;
  const long long smem = policy_smem_bytes(n, C);
  if (smem > kPolSmemMax) return set_error(MS_ERR_INVALID, "policy_apply: queue too long for the per-job tables");
  if (!lat_us || !credit || !acc || !n_cand || !deadline_us || !assigned || !ws || !status)
    return set_error(MS_ERR_INVALID, "policy_apply: null pointer");
  if (!(factor > 0.0) || grid_us < 1) return set_error(MS_ERR_INVALID, "policy_apply: factor > 0, grid_us >= 1");
  const long long cells = ws_bytes / 16;  // one int64 value + one double per cell
  if (cells < 2LL * n + 2) return set_error(MS_ERR_INVALID, "policy_apply: workspace too small");
  long long* hval = reinterpret_cast<long long*>(ws);
  double* hworst = reinterpret_cast<double*>(hval + cells);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(policy_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPolSmemMax);
    attr = true;
  }
  policy_apply_kernel<<<1, kPolThreads, (size_t)smem, reinterpret_cast<cudaStream_t>(stream)>>>(
      n, C, reinterpret_cast<const long long*>(lat_us), credit, acc, n_cand,
      reinterpret_cast<const long long*>(deadline_us), assigned, now_us, running_finish_us, has_running, factor,
      grid_us, hval, hworst, cells, status);
  return check_launch("policy_apply_kernel");
}

int ms_policy_max_jobs(int C) {
  if (C < 1 || C > 64) return 0;
  int n = 1;
  while (policy_smem_bytes(n + 1, C) <= kPolSmemMax) ++n;
  return n;
}

}  // extern "C"
