// FP64 peak microbenchmark for B200 (sm_100a): DMMA (mma.sync f64) and DFMA
// throughput, burst and sustained, plus a layout self-check of the f64 mma
// fragment mappings the GEMM kernels rely on.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peaks fp64_peaks.cu
// Output: one JSON object on stdout (MEASURED_FP64.json).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cmath>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ void mma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ void mma16816(double (&d)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 "
               "{%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                 "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

// 8 independent accumulator chains per warp to cover DMMA latency.
template <int CHAINS>
__global__ void dmma884_loop(double* out, long iters) {
  double acc[CHAINS][2];
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c][0] = acc[c][1] = 0.0;
  for (long i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) mma884(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c][0] + acc[c][1];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void dmma16816_loop(double* out, long iters) {
  double acc[CHAINS][4];
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + (threadIdx.x + i) * 1e-9;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - (threadIdx.x + i) * 1e-9;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c][0] = acc[c][1] = acc[c][2] = acc[c][3] = 0.0;
  for (long i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) mma16816(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c][0] + acc[c][1] + acc[c][2] + acc[c][3];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void dfma_loop(double* out, long iters) {
  double acc[CHAINS];
  double a = 1.0 + threadIdx.x * 1e-12, b = 1e-9;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = c;
  for (long i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

// Layout self-check: D = A*B with A 16x16 row-major, B 16x8 (B[k][n]) through
// m16n8k16 and through 4x m8n8k4 on the same data.
__global__ void layout_check(const double* A, const double* B, double* D16, double* D8) {
  int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a[8], b[4], d[4] = {0, 0, 0, 0};
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = A[(g + 8 * (i & 1)) * 16 + (t + 4 * (i >> 1))];
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = B[(t + 4 * i) * 8 + g];
  mma16816(d, a, b);
  D16[g * 8 + 2 * t] = d[0];
  D16[g * 8 + 2 * t + 1] = d[1];
  D16[(g + 8) * 8 + 2 * t] = d[2];
  D16[(g + 8) * 8 + 2 * t + 1] = d[3];
  // m8n8k4: rows 0..7 and 8..15 separately, k in steps of 4
  for (int mh = 0; mh < 2; ++mh) {
    double c[2] = {0, 0};
    for (int k0 = 0; k0 < 16; k0 += 4) {
      double av = A[(mh * 8 + g) * 16 + k0 + t];
      double bv = B[(k0 + t) * 8 + g];
      mma884(c, av, bv);
    }
    D8[(mh * 8 + g) * 8 + 2 * t] = c[0];
    D8[(mh * 8 + g) * 8 + 2 * t + 1] = c[1];
  }
}

__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) b[i] = a[i];
}

template <typename K>
static double time_kernel(K kern, int grid, int block, long iters, int reps, double* out) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  kern<<<grid, block>>>(out, iters / 10 + 1);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(e0));
    kern<<<grid, block>>>(out, iters);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount;
  double* out;
  CK(cudaMalloc(&out, 64));

  // layout check
  {
    std::vector<double> A(256), B(128), D16(128), D8(128), R(128, 0.0);
    for (int i = 0; i < 256; ++i) A[i] = (i * 37 % 101) * 0.01 - 0.5;
    for (int i = 0; i < 128; ++i) B[i] = (i * 53 % 97) * 0.01 - 0.4;
    for (int m = 0; m < 16; ++m)
      for (int n = 0; n < 8; ++n)
        for (int k = 0; k < 16; ++k) R[m * 8 + n] += A[m * 16 + k] * B[k * 8 + n];
    double *dA, *dB, *dD16, *dD8;
    CK(cudaMalloc(&dA, 256 * 8)); CK(cudaMalloc(&dB, 128 * 8));
    CK(cudaMalloc(&dD16, 128 * 8)); CK(cudaMalloc(&dD8, 128 * 8));
    CK(cudaMemcpy(dA, A.data(), 256 * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), 128 * 8, cudaMemcpyHostToDevice));
    layout_check<<<1, 32>>>(dA, dB, dD16, dD8);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(D16.data(), dD16, 128 * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(D8.data(), dD8, 128 * 8, cudaMemcpyDeviceToHost));
    double e16 = 0, e8 = 0;
    for (int i = 0; i < 128; ++i) {
      e16 = fmax(e16, fabs(D16[i] - R[i]));
      e8 = fmax(e8, fabs(D8[i] - R[i]));
    }
    fprintf(stderr, "layout check: m16n8k16 maxerr %.3e, m8n8k4 maxerr %.3e\n", e16, e8);
    printf("{\"layout_err_m16n8k16\": %.3e, \"layout_err_m8n8k4\": %.3e,\n", e16, e8);
  }

  const long iters = 20000;
  const int reps = 5;
  // DMMA m8n8k4: per warp-instruction 8*8*4 FMA = 512 flop
  double best884 = 0;
  int best_warps = 0;
  for (int warps : {4, 8, 16}) {
    int grid = sms * 2, block = 32 * warps;
    double ms = time_kernel(dmma884_loop<8>, grid, block, iters, reps, out);
    double flops = (double)grid * warps * iters * 8 * 512.0;
    double tf = flops / (ms * 1e-3) / 1e12;
    fprintf(stderr, "DMMA m8n8k4 warps/CTA=%d: %.2f TFLOP/s\n", warps, tf);
    if (tf > best884) { best884 = tf; best_warps = warps; }
  }
  double best16 = 0;
  for (int warps : {4, 8}) {
    int grid = sms * 2, block = 32 * warps;
    double ms = time_kernel(dmma16816_loop<4>, grid, block, iters / 4, reps, out);
    double flops = (double)grid * warps * (iters / 4) * 4 * (16.0 * 8 * 16 * 2);
    double tf = flops / (ms * 1e-3) / 1e12;
    fprintf(stderr, "DMMA m16n8k16 warps/CTA=%d: %.2f TFLOP/s\n", warps, tf);
    if (tf > best16) best16 = tf;
  }
  double bestfma = 0;
  for (int warps : {8, 16, 32}) {
    int grid = sms * 2, block = 32 * warps;
    double ms = time_kernel(dfma_loop<8>, grid, block, iters, reps, out);
    double flops = (double)grid * block * iters * 8 * 2.0;
    double tf = flops / (ms * 1e-3) / 1e12;
    fprintf(stderr, "DFMA warps/CTA=%d: %.2f TFLOP/s\n", warps, tf);
    if (tf > bestfma) bestfma = tf;
  }
  // sustained DMMA: back-to-back for ~4 s
  double sustained = 0;
  {
    int grid = sms * 2, block = 32 * best_warps;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    double ms_one = time_kernel(dmma884_loop<8>, grid, block, iters, 1, out);
    int n = (int)(4000.0 / ms_one) + 1;
    CK(cudaEventRecord(e0));
    for (int i = 0; i < n; ++i) dmma884_loop<8><<<grid, block>>>(out, iters);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    double flops = (double)n * grid * best_warps * iters * 8 * 512.0;
    sustained = flops / (ms * 1e-3) / 1e12;
    fprintf(stderr, "DMMA sustained (%d launches, %.0f ms): %.2f TFLOP/s\n", n, ms, sustained);
  }
  // HBM copy (double2), 4 GiB read + 4 GiB write
  double copy_gbs = 0;
  {
    size_t bytes = (size_t)4 << 30;
    size_t n = bytes / 16;
    double2 *a, *b;
    CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes));
    CK(cudaMemset(a, 0, bytes));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    float best = 1e30f;
    for (int r = 0; r < 6; ++r) {
      CK(cudaEventRecord(e0));
      copy_kernel<<<sms * 8, 512>>>(a, b, n);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (r > 0 && ms < best) best = ms;
    }
    copy_gbs = 2.0 * bytes / (best * 1e-3) / 1e9;
    fprintf(stderr, "HBM copy: %.1f GB/s\n", copy_gbs);
    cudaFree(a); cudaFree(b);
  }
  printf(" \"gpu_name\": \"%s\", \"sms\": %d,\n", prop.name, sms);
  printf(" \"dmma_m8n8k4_tflops\": %.3f, \"dmma_m16n8k16_tflops\": %.3f, \"dfma_tflops\": %.3f,\n",
         best884, best16, bestfma);
  printf(" \"dmma_sustained_tflops\": %.3f, \"copy_fp64_gbs\": %.1f}\n", sustained, copy_gbs);
  return 0;
}
