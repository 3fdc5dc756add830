// Coupled queue policy on the device: the reference's
// OPTIMIZED dropping policy over a whole EDF queue,
//
//   apply_policy(OPTIMIZED)          scheduler.py:382-425
//     detect_violation / budget      scheduler.py:187-233 (prefix sums of est)
//     reassign_optimized (MCKP)      scheduler.py:236-326 (grid DP + reconstruction)
//     try_upgrade                    scheduler.py:366-379
//
// in ONE single-CTA launch.  Control flow (violation search, budget, drops,
// reconstruction, upgrades) runs on thread 0; the knapsack's value/accuracy
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
constexpr int kPolMaxJobs = 1024;
constexpr int kPolMaxUnits = 4096;  // jobs x candidates (shared grid-unit table)

__device__ __forceinline__ long long est_us(long long lat, double f) {
  return __double2ll_rn((double)lat * f);  // Python round(): half-even
}
__device__ __forceinline__ long long floordiv(long long a, long long b) {  // b > 0
  long long q = a / b;
  if ((a % b) != 0 && a < 0) --q;
  return q;
}

__global__ void __launch_bounds__(kPolThreads) policy_apply_kernel(
    int n, int C, const long long* __restrict__ lat, const int32_t* __restrict__ credit,
    const double* __restrict__ acc, const int32_t* __restrict__ n_cand, const long long* __restrict__ deadline,
    int32_t* __restrict__ assigned_io, long long now_us, long long running_finish_us, int has_running,
    double factor, long long grid_us, long long* __restrict__ hval, double* __restrict__ hworst,
    long long hist_cells, int32_t* __restrict__ status) {
  __shared__ int32_t s_asg[kPolMaxJobs];
  __shared__ uint8_t s_alive[kPolMaxJobs];
  __shared__ int32_t s_scope[kPolMaxJobs];
  __shared__ long long s_caps[kPolMaxJobs];
  __shared__ int32_t s_units[kPolMaxUnits];
  __shared__ int s_m, s_width, s_v, s_phase;
  __shared__ long long s_best_val[kPolThreads / 32];
  __shared__ double s_best_w[kPolThreads / 32];
  __shared__ int s_best_t[kPolThreads / 32];

  const int tid = threadIdx.x;
  if (tid == 0) *status = 0;
  for (int j = tid; j < n; j += blockDim.x) {
    s_asg[j] = assigned_io[j];
    s_alive[j] = 1;
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
        if (!s_alive[j]) continue;
        t += est_us(lat[(long long)j * C + s_asg[j]], factor);
        if (t > deadline[j]) {
          v = j;
          break;
        }
      }
      s_v = v;
      s_phase = 0;  // 0: stop, 1: drop v, 2: run the knapsack
      if (v >= 0) {
        const long long budget = deadline[v] - dispatch;  // compute_budget (start = dispatch)
        s_phase = 1;
        if (budget > 0) {
          // scope = queued jobs up to and including v; grid units and prefix caps
          int m = 0;
          long long run = 0, min_cap = 0;
          bool ok = true;
          for (int j = 0; j <= v && ok; ++j) {
            if (!s_alive[j]) continue;
            if ((m + 1) * C > kPolMaxUnits) {
              ok = false;
              *status = 2;
              break;
            }
            long long mx = 0;
            for (int c = 0; c < n_cand[j]; ++c) {
              const long long e = est_us(lat[(long long)j * C + c], factor);
              const long long u = (e + grid_us - 1) / grid_us;  // e >= 0: -(-e // grid)
              s_units[m * C + c] = (int32_t)u;
              mx = u > mx ? u : mx;
            }
            run += mx;
            long long cap = budget / grid_us;
            cap = run < cap ? run : cap;
            const long long dl = floordiv(deadline[j] - dispatch, grid_us);
            cap = dl < cap ? dl : cap;
            s_caps[m] = cap;
            min_cap = (m == 0 || cap < min_cap) ? cap : min_cap;
            s_scope[m++] = j;
          }
          if (ok && min_cap >= 0) {
            const long long width = s_caps[m - 1] + 1;
            if (width * (long long)(m + 1) > hist_cells) {
              *status = 1;  // workspace too small: caller falls back to the host policy
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
        const int j = s_scope[i];
        const long long* pv = hval + (long long)i * width;
        const double* pw = hworst + (long long)i * width;
        long long* nv = hval + (long long)(i + 1) * width;
        double* nw = hworst + (long long)(i + 1) * width;
        const long long top = min(s_caps[i], (long long)width - 1);
        const int nc = n_cand[j];
        for (int t = tid; t < width; t += blockDim.x) {
          long long dv = -1;
          double dw = -INFINITY;
          if (t <= top) {
            for (int c = 0; c < nc; ++c) {
              const int d = s_units[i * C + c];
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
      if ((tid & 31) == 0) {
        s_best_val[tid >> 5] = bv;
        s_best_w[tid >> 5] = bw;
        s_best_t[tid >> 5] = bt;
      }
      __syncthreads();
      if (tid == 0) {
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
          s_alive[s_v] = 0;  // no feasible assignment: drop the violator
        } else {
          // reconstruction from the back: the fastest (first) candidate that
          // reproduces the optimum at each step
          long long want_v = bv;
          double want_w = bw;
          int t = bt;
          for (int i = m - 1; i >= 0; --i) {
            const int j = s_scope[i];
            const long long* pv = hval + (long long)i * width;
            const double* pw = hworst + (long long)i * width;
            for (int c = 0; c < n_cand[j]; ++c) {
              const int d = s_units[i * C + c];
              const int s = t - d;
              if (s < 0 || t > s_caps[i] || pv[s] < 0) continue;
              const double a = acc[(long long)j * C + c];
              const double mw = pw[s] < a ? pw[s] : a;
              if (pv[s] + credit[(long long)j * C + c] == want_v && mw == want_w) {
                s_asg[j] = c;
                t = s;
                want_v = pv[s];
                want_w = pw[s];
                break;
              }
            }
          }
        }
      }
      __syncthreads();
    } else {  // phase 1: budget <= 0 or infeasible caps -> drop the violator
      if (tid == 0) s_alive[s_v] = 0;
      __syncthreads();
    }
  }

  // ----------------------------------------------------------- try_upgrade
  if (tid == 0) {
    // completion times and suffix-min slack over the queued jobs (no violation)
    long long* comp = hval;       // reuse the workspace: [n]
    long long* sfx = hval + n;    // suffix min of deadline - completion
    long long t = dispatch;
    for (int j = 0; j < n; ++j) {
      if (!s_alive[j]) continue;
      t += est_us(lat[(long long)j * C + s_asg[j]], factor);
      comp[j] = t;
    }
    auto rebuild = [&]() {
      long long mn = LLONG_MAX;
      for (int j = n - 1; j >= 0; --j) {
        if (s_alive[j]) {
          const long long sl = deadline[j] - comp[j];
          mn = sl < mn ? sl : mn;
        }
        sfx[j] = mn;
      }
    };
    rebuild();
    bool moved = true;
    while (moved) {
      moved = false;
      for (int j = 0; j < n; ++j) {
        if (!s_alive[j]) continue;
        while (s_asg[j] + 1 < n_cand[j]) {
          const long long old_e = est_us(lat[(long long)j * C + s_asg[j]], factor);
          const long long new_e = est_us(lat[(long long)j * C + s_asg[j] + 1], factor);
          const long long delta = new_e - old_e;
          if (delta > sfx[j]) break;  // would create a violation at or after j
          s_asg[j] += 1;
          moved = true;
          if (delta != 0) {
            for (int k = j; k < n; ++k)
              if (s_alive[k]) comp[k] += delta;
            rebuild();
          }
        }
      }
    }
  }
  __syncthreads();
  for (int j = tid; j < n; j += blockDim.x) assigned_io[j] = s_alive[j] ? s_asg[j] : -1;
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
  if (n > kPolMaxJobs) return set_error(MS_ERR_INVALID, "policy_apply: at most 1024 queued jobs");
  if (!lat_us || !credit || !acc || !n_cand || !deadline_us || !assigned || !ws || !status)
    return set_error(MS_ERR_INVALID, "policy_apply: null pointer");
  if (!(factor > 0.0) || grid_us < 1) return set_error(MS_ERR_INVALID, "policy_apply: factor > 0, grid_us >= 1");
  const long long cells = ws_bytes / 16;  // one int64 value + one double per cell
  if (cells < 2LL * n + 2) return set_error(MS_ERR_INVALID, "policy_apply: workspace too small");
  long long* hval = reinterpret_cast<long long*>(ws);
  double* hworst = reinterpret_cast<double*>(hval + cells);
  policy_apply_kernel<<<1, kPolThreads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      n, C, reinterpret_cast<const long long*>(lat_us), credit, acc, n_cand,
      reinterpret_cast<const long long*>(deadline_us), assigned, now_us, running_finish_us, has_running, factor,
      grid_us, hval, hworst, cells, status);
  return check_launch("policy_apply_kernel");
}

}  // extern "C"
