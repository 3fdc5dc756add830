// Error plumbing shared by the C-ABI entry points.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "mosel_b200.h"

namespace mosel {
int set_error(int code, const char* msg);
int check_launch(const char* what);
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
