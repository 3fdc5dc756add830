// Offline strategy DP on the device: the reference's exact
// min-latency table over (requests covered r, accuracy credit c)
// (strategy.py:139-177 _DpTables; host mirror planner._Table).
//
//   lat[r, c] = min over items (mask, batch b, latency L, credit index ci)
//               with b <= r, ci <= c, c < r*unit+1 of  lat[r-b, c-ci] + L
//   cnt[r, c] = least part count among the latency-minimal candidates
//
// The reference relaxes one item at a time over a numpy slice; the final
// (lat, cnt) of every cell is the lexicographic minimum over its candidates
// (a better latency always replaces both; an equal latency can only lower
// the count), so evaluating each cell independently over all items gives
// the identical table.  Row r depends only on rows < r: one launch per row,
// one thread per credit cell.  The host keeps the reference's query and
// back-walk (planner._Table.query / _walk) on the downloaded table, so
// matrices are byte-identical (tests/golden/matrices).  S=128 tables that
// take the numpy reference minutes build in milliseconds here.
#include <cstdint>

#include "mosel_b200.h"
#include "ptx.cuh"
#include "runtime.h"

namespace mosel {

constexpr long long kDpBig = 1LL << 62;
constexpr int kDpPartsBig = 0x7fffffff;

__global__ void __launch_bounds__(256) strategy_dp_row_kernel(int r, long long width, long long limit, int n_items,
                                                              const int32_t* __restrict__ batch,
                                                              const long long* __restrict__ lat_us,
                                                              const int32_t* __restrict__ cidx,
                                                              long long* __restrict__ lat,
                                                              int32_t* __restrict__ cnt) {
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < limit;
       c += (long long)gridDim.x * blockDim.x) {
    long long best = kDpBig;
    int best_n = kDpPartsBig;
    for (int i = 0; i < n_items; ++i) {
      const int b = batch[i];
      const int ci = cidx[i];
      if (b > r || ci > c) continue;
      const long long src = lat[(long long)(r - b) * width + (c - ci)];
      if (src >= kDpBig) continue;  // unreachable source (never selected by the reference)
      const long long cand = src + lat_us[i];
      const int cand_n = cnt[(long long)(r - b) * width + (c - ci)] + 1;
      if (cand < best || (cand == best && cand_n < best_n)) {
        best = cand;
        best_n = cand_n;
      }
    }
    lat[(long long)r * width + c] = best;
    cnt[(long long)r * width + c] = best_n;
  }
}

__global__ void strategy_dp_init_kernel(long long cells, long long* __restrict__ lat, int32_t* __restrict__ cnt) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < cells;
       i += (long long)gridDim.x * blockDim.x) {
    lat[i] = i == 0 ? 0 : kDpBig;
    cnt[i] = i == 0 ? 0 : kDpPartsBig;
  }
}

}  // namespace mosel

using namespace mosel;

extern "C" {

int ms_strategy_dp(int n_items, const int32_t* batch, const int64_t* lat_us, const int32_t* credit_idx, int max_size,
                   int unit, int64_t* lat, int32_t* cnt, void* stream) {
  if (n_items < 1 || max_size < 0 || unit < 0) return set_error(MS_ERR_INVALID, "strategy_dp: bad shape");
  if (!batch || !lat_us || !credit_idx || !lat || !cnt) return set_error(MS_ERR_INVALID, "strategy_dp: null pointer");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const long long width = (long long)max_size * unit + 1;
  const long long cells = (long long)(max_size + 1) * width;
  long long blocks = (cells + 255) / 256;
  if (blocks > 148LL * 16) blocks = 148LL * 16;
  strategy_dp_init_kernel<<<(int)blocks, 256, 0, st>>>(cells, reinterpret_cast<long long*>(lat), cnt);
  int rc = check_launch("strategy_dp_init_kernel");
  if (rc) return rc;
  for (int r = 1; r <= max_size; ++r) {
    const long long limit = (long long)r * unit + 1;
    long long rb = (limit + 255) / 256;
    if (rb > 148LL * 16) rb = 148LL * 16;
    strategy_dp_row_kernel<<<(int)rb, 256, 0, st>>>(r, width, limit, n_items, batch,
                                                     reinterpret_cast<const long long*>(lat_us), credit_idx,
                                                     reinterpret_cast<long long*>(lat), cnt);
    rc = check_launch("strategy_dp_row_kernel");
    if (rc) return rc;
  }
  return MS_OK;
}

}  // extern "C"
