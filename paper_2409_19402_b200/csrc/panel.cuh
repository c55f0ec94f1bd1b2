// Small-panel kernels of the batched subspace iteration (panel.cu).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace ppc {

// split-K chunk count of a panel with r rows (128 rows per chunk)
int panel_splits(int64_t r);
// the kernels take panels of bc <= 64 columns and r >= 128 rows
bool panel_kernels_ok(int64_t r, int64_t bc);
// S (bc x bc per slice at S + slice*bc*bc, full symmetric) = A^T B for the
// r x bc panels A (stride sA per slice) and B (sB), the upper triangle
// mirrored (A^T B is symmetric for the callers: Y^T Y, X^T G X); batch
// launch slots, slot z -> slice zmap[z] (nullable).
// part: workspace of panel_splits(r) * max(zext, batch) * bc * bc doubles.
void panel_gram(const double* A, int64_t sA, const double* B, int64_t sB, int64_t r, int64_t bc, int64_t batch,
                double* S, double* part, int64_t zext, const int* zmap, cudaStream_t s);
// Rinv (bc x bc per slice, upper, zeros below) = R^{-1} with R^T R = S (+ a
// 1e-15 trace shift); fail: non-positive pivot; weak (nullable, per slice):
// a pivot below 1e-12 of the largest diagonal.
void chol_inv64(const double* S, int64_t bc, int64_t batch, bool shift, double* Rinv, int* fail, const int* zmap,
                int* weak, cudaStream_t s);
// Yout (r x bc per slice) = Yin * M (bc x bc per slice, column-major).
void panel_apply(const double* Yin, int64_t sIn, const double* M, double* Yout, int64_t sOut, int64_t r, int64_t bc,
                 int64_t batch, const int* zmap, cudaStream_t s);

}  // namespace ppc
