// Error plumbing shared by the C-ABI entry points.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "mosel_b200.h"

#include <utility>

namespace mosel {
int set_error(int code, const char* msg);
int check_launch(const char* what);

// Programmatic dependent launch for the op-program kernels (ms_set_pdl).
extern int g_pdl;

// cudaLaunchKernelEx with the PDL attribute (when enabled) and an optional
// cluster dimension.  Every kernel launched through here calls pdl_wait()
// before its first dependent global access.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            int cluster_x, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int n = 0;
  if (cluster_x > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster_x;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  if (g_pdl) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
// gemm.cu: cuTensorMapEncodeTiled for a bf16 tensor (driver entry point)
int encode_bf16_map(CUtensorMap* m, int rank, const void* base, const cuuint64_t* dims, const cuuint64_t* strides_bytes,
                    const cuuint32_t* box, const cuuint32_t* estride, CUtensorMapSwizzle swz);
// transformer.cu
int run_layernorm(const void* X, long long ldx, long long rows, const float* gamma, const float* beta, void* Y,
                  long long ldy, int C, float eps, cudaStream_t st);
int run_attention(const void* qkv, long long ld, int L, int H, int n_seq, void* out, long long ldo, float scale,
                  cudaStream_t st);
int run_patchify(const void* X, int n, int S, int C, int P, void* Y, cudaStream_t st);
int run_vit_embed(const void* pe, const void* cls, const void* pos, int n, int L, int D, void* tok, cudaStream_t st);
int run_bert_embed(const int32_t* ids, long long n_tok, int L, const void* word, const void* pos, const void* type0,
                   const float* gamma, const float* beta, void* Y, int D, float eps, cudaStream_t st);
}  // namespace mosel
