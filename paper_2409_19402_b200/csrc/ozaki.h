// FP64 Gram on the INT8 tensor cores (Ozaki scheme, ozaki.cu).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace ppc {

// Per-plan-chunk partial Grams parts[c] = T_c^T T_c (nchunks x n3 x n3) of a
// tube matrix T (rows x n3, leading dimension ldT), as gram_partials, through
// 7-digit int8 splitting and tcgen05 kind::i8 MMAs. Returns false when the
// shape is not eligible (caller falls back to the DMMA SYRK). PPC_OZAKI=0
// disables it.
bool ozaki_gram_partials(const double* T, int64_t ldT, int64_t rows, int64_t n3, int64_t chunk, int64_t nchunks,
                         double* parts, cudaStream_t s);

// G_b (n x n, column-major, b < batch, stride n*n) = A_b^T A_b for A_b
// (rows x n, leading dimension lda) at A + b*strideA: the batched slice
// Grams. rows <= 65536. Returns false when not eligible.
bool ozaki_syrk_batched(const double* A, int64_t lda, int64_t strideA, int64_t rows, int64_t n, int64_t batch,
                        double* G, cudaStream_t s);

}  // namespace ppc
