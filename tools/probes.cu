// Debug probes for tools/umma_probe.py and tools/umma_rate.py (NOT part of
// the product library): UMMA shifted-descriptor behaviour and raw tcgen05.mma
// issue rates.  Built on demand by tools/_probes.py into tools/_probes.so.
#include <cstdint>

#include "mosel_b200.h"
#include "ptx.cuh"

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static int encode_map(CUtensorMap* m, int rank, const void* base, const cuuint64_t* dims, const cuuint64_t* strides,
                      const cuuint32_t* box, const cuuint32_t* es,
                      CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  void* ptr = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) != cudaSuccess) return 1;
  return reinterpret_cast<EncodeFn>(ptr)(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), dims,
                                         strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != 0;
}
static int check_launch(const char*) { return cudaGetLastError() == cudaSuccess ? 0 : 1; }

namespace mosel {
constexpr int kBK = 64;
}  // namespace mosel


// ------------------------------------------------------------------------
// Debug probe (tools/umma_probe.py): does a K-major SW128 A descriptor whose
// start address is shifted by `shift` 128-byte rows (with the descriptor's
// base-offset field = shift & 7, and an explicit SBO) read rows
// [shift, shift + 128) of a TMA-written tile?  This is the addressing a
// halo-reusing 3x3 conv needs (taps = shifted windows of one smem tile).
namespace mosel {
__global__ void __launch_bounds__(128, 1) umma_shift_probe_kernel(const __grid_constant__ CUtensorMap tmA,
                                                                  const __grid_constant__ CUtensorMap tmB,
                                                                  float* D, int shift, int sbo, int use_base) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;                 // 256 rows x 128 B
  uint8_t* sB = smem + 256 * 128;     // 64 rows x 128 B
  __shared__ uint64_t bar, mbar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&mbar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&tslot, 64);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tslot;
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, 256 * 128 + 64 * 128);
    tma_load_2d(smem_addr(sA), &tmA, &bar, 0, 0);
    tma_load_2d(smem_addr(sA + 128 * 128), &tmA, &bar, 0, 128);
    tma_load_2d(smem_addr(sB), &tmB, &bar, 0, 0);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t a_addr = smem_addr(sA) + (uint32_t)shift * 128u;
    uint64_t adesc = 0;
    adesc |= (uint64_t)((a_addr & 0x3FFFF) >> 4);
    adesc |= (uint64_t)1 << 16;
    adesc |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    adesc |= (uint64_t)1 << 46;
    if (use_base) adesc |= (uint64_t)((a_addr >> 7) & 7) << 49;
    adesc |= (uint64_t)2 << 61;
    const uint64_t bdesc = umma_desc_sw128(smem_addr(sB));
    const uint32_t idesc = umma_idesc_bf16_m128(64);
    for (int k = 0; k < 4; ++k) umma_bf16(tb, adesc + 2 * k, bdesc + 2 * k, idesc, k != 0);
    umma_commit(&mbar);
  }
  mbar_wait(&mbar, 0);
  tc_fence_after();
  for (int c = 0; c < 2; ++c) {
    uint32_t v[32];
    tmem_ld_32x32b_x32(tb + (uint32_t)(c * 32) + ((uint32_t)(warp * 32) << 16), v);
    tmem_wait_ld();
    for (int j = 0; j < 32; ++j) D[(warp * 32 + lane) * 64 + c * 32 + j] = __uint_as_float(v[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tb, 64);
}
}  // namespace mosel

extern "C" int ms_debug_umma_shift(const void* A /* [256, 64] bf16 */, const void* W /* [64, 64] bf16 */,
                                   float* D /* [128, 64] */, int shift, int sbo, int use_base, void* stream) {
  using namespace mosel;
  CUtensorMap ta, tb;
  cuuint64_t da[2] = {64, 256}, sa[1] = {128};
  cuuint32_t ba[2] = {64, 128}, es[2] = {1, 1};
  int rc = encode_map(&ta, 2, A, da, sa, ba, es);
  if (rc) return rc;
  cuuint64_t db[2] = {64, 64}, sb[1] = {128};
  cuuint32_t bb[2] = {64, 64};
  rc = encode_map(&tb, 2, W, db, sb, bb, es);
  if (rc) return rc;
  cudaFuncSetAttribute(umma_shift_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  umma_shift_probe_kernel<<<1, 128, 50 * 1024, reinterpret_cast<cudaStream_t>(stream)>>>(ta, tb, D, shift, sbo,
                                                                                           use_base);
  return check_launch("umma_shift_probe_kernel");
}

// ------------------------------------------------------------------------
// Debug probe (tools/umma_rate.py): issue rate of back-to-back
// tcgen05.mma (M=128, K=16) from one thread into one accumulator, for an A
// descriptor of layout `mode` (0 = SW128 K-major, 1 = no-swizzle LBO 16 /
// SBO 128, 2 = no-swizzle LBO 16 / SBO 112, 3 = no-swizzle LBO 128 / SBO 256
// canonical) and width n.  Operands are uninitialised shared memory: only the
// timing is meaningful.  cycles[0] = clocks from the first issue to the
// commit's completion.
namespace mosel {
__global__ void __launch_bounds__(128, 1) umma_rate_kernel(int mode, int n, int count, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t mbar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&mbar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&tslot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tslot;
  if (threadIdx.x == 0) {
    const uint32_t a0 = smem_addr(smem), b0 = smem_addr(smem + 64 * 1024);
    uint64_t ad;
    // mode 4 + r: SW128 starting r 128-B rows into the tile (halo tap views);
    // mode 20 / 21: the 9 tap shifts of a halo of pitch 16 / 32, rotating
    const int pitch = mode == 20 ? 16 : 32;
    uint64_t tap_desc[9];
    for (int t = 0; t < 9; ++t) tap_desc[t] = umma_desc_sw128(a0 + (uint32_t)(((t / 3) * pitch + t % 3) * 128));
    if (mode >= 20) {
      const uint64_t bd = umma_desc_sw128(b0);
      const uint32_t idesc = umma_idesc_bf16_m128((uint32_t)n);
      const long long t0 = clock64();
      for (int i = 0; i < count; ++i) umma_bf16(tb, tap_desc[(i >> 2) % 9] + 2 * (i & 3), bd + 2 * (i & 3), idesc, i != 0);
      umma_commit(&mbar);
      mbar_wait(&mbar, 0);
      cycles[0] = clock64() - t0;
    } else {
    if (mode >= 4) ad = umma_desc_sw128(a0 + (uint32_t)(mode - 4) * 128u);
    else if (mode == 0) ad = umma_desc_sw128(a0);
    else if (mode == 1) ad = umma_desc_interleave(a0, 16, 128);
    else if (mode == 2) ad = umma_desc_interleave(a0, 16, 112);
    else ad = umma_desc_interleave(a0, 128, 256);
    const uint64_t bd = umma_desc_sw128(b0);
    const uint32_t idesc = umma_idesc_bf16_m128((uint32_t)n);
    const long long t0 = clock64();
    for (int i = 0; i < count; ++i) umma_bf16(tb, ad + 2 * (i & 3), bd + 2 * (i & 3), idesc, i != 0);
    umma_commit(&mbar);
    mbar_wait(&mbar, 0);
    cycles[0] = clock64() - t0;
    }
  }
  __syncthreads();
  if (warp == 0) tmem_dealloc(tb, 256);
}
}  // namespace mosel

extern "C" int ms_debug_umma_rate(int mode, int n, int count, long long* cycles, void* stream) {
  using namespace mosel;
  cudaFuncSetAttribute(umma_rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  umma_rate_kernel<<<1, 128, 150 * 1024, reinterpret_cast<cudaStream_t>(stream)>>>(mode, n, count, cycles);
  return check_launch("umma_rate_kernel");
}
