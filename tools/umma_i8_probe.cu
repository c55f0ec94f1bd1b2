// Probe: tcgen05 kind::i8 GEMM with TMA (128B swizzle) + TMEM accumulators.
// C[M x N] (int32, row-major) = A[M x K] (int8, K contiguous) * B[N x K]^T.
// Checks a sample of entries against a CPU reference and reports TOPS.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2409_19402_b200/csrc \
//        tools/umma_i8_probe.cu -o tools/umma_i8_probe
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "umma_i8.cuh"

using namespace ppc::umma;

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e = (x);                                                                   \
        if (e != cudaSuccess) {                                                                \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
            exit(1);                                                                           \
        }                                                                                      \
    } while (0)

constexpr int BM = 128, BK = 128;

template <int BN, int STAGES>
__global__ void __launch_bounds__(192, 1)
    i8_gemm_probe(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb, int32_t* C, int M,
                  int N, int K) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* As = base;
    uint8_t* Bs = base + STAGES * BM * BK;
    uint64_t* full = reinterpret_cast<uint64_t*>(Bs + STAGES * BN * BK);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(tfull + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int mt = blockIdx.x, nt = blockIdx.y;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            bar_init(&full[s], 1);
            bar_init(&empty[s], 1);
        }
        bar_init(tfull, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<BN>(tslot);
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tmem = *tslot;
    const int nk = K / BK;
    if (warp == 0) {
        if (elect_one()) {
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % STAGES;
                bar_wait(&empty[s], ((kb / STAGES) & 1) ^ 1);
                bar_expect_tx(&full[s], (BM + BN) * BK);
                tma_load_2d(As + s * BM * BK, &ma, &full[s], kb * BK, mt * BM);
                tma_load_2d(Bs + s * BN * BK, &mb, &full[s], kb * BK, nt * BN);
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idesc = idesc_i8<BM, BN>();
        for (int kb = 0; kb < nk; ++kb) {
            const int s = kb % STAGES;
            bar_wait(&full[s], (kb / STAGES) & 1);
            fence_after_sync();
            if (elect_one()) {
                const uint64_t da = sdesc_k_sw128(As + s * BM * BK);
                const uint64_t db = sdesc_k_sw128(Bs + s * BN * BK);
#pragma unroll
                for (int kk = 0; kk < BK / 32; ++kk)
                    mma_i8(tmem, da + (uint64_t)(kk * 2), db + (uint64_t)(kk * 2), idesc, (kb | kk) != 0);
                mma_commit(&empty[s]);
            }
            __syncwarp();
        }
        if (elect_one()) mma_commit(tfull);
        __syncwarp();
    } else {
        bar_wait(tfull, 0);
        fence_after_sync();
        const int q = warp & 3;
        const int row = mt * BM + q * 32 + lane;
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
            int32_t v[32];
            tmem_ld_32x32b_x32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c, v);
            tmem_ld_wait();
            int32_t* dst = C + (size_t)row * N + nt * BN + c;
#pragma unroll
            for (int j = 0; j < 32; j += 4) *reinterpret_cast<int4*>(dst + j) = make_int4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        }
    }
    fence_before_sync();
    __syncthreads();
    if (warp == 1) tmem_free<BN>(tmem);
}

// MN-major A variant: A stored [K][M] (M contiguous), SWIZZLE_64B tiles of
// 64 M-bytes x 64 K-rows (8-row K groups SBO = 512 B apart, 64-byte M atoms
// LBO apart); B K-major SWIZZLE_64B; BM = 128, BN = 64, BK = 64.
__device__ __forceinline__ uint64_t sdesc_mn_sw64(const void* smem_tile, uint32_t lbo_bytes) {
    const uint32_t a = smem_u32(smem_tile);
    uint64_t d = 0;
    d |= (uint64_t)((a >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)(512 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)4 << 61;
    return d;
}

__global__ void __launch_bounds__(192, 1)
    i8_gemm_mn_probe(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb, int32_t* C, int M,
                     int N, int K) {
    constexpr int BMm = 128, BNn = 64, BKk = 64, ST = 4;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* As = base;                         // ST x (2 x 4096)
    uint8_t* Bs = base + ST * BMm * BKk;        // ST x 4096
    uint64_t* full = reinterpret_cast<uint64_t*>(Bs + ST * BNn * BKk);
    uint64_t* empty = full + ST;
    uint64_t* tfull = empty + ST;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(tfull + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int mt = blockIdx.x, nt = blockIdx.y;
    if (threadIdx.x == 0) {
        for (int s = 0; s < ST; ++s) {
            bar_init(&full[s], 1);
            bar_init(&empty[s], 1);
        }
        bar_init(tfull, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<64>(tslot);
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tmem = *tslot;
    const int nk = K / BKk;
    if (warp == 0) {
        if (elect_one()) {
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % ST;
                bar_wait(&empty[s], ((kb / ST) & 1) ^ 1);
                bar_expect_tx(&full[s], (BMm + BNn) * BKk);
                tma_load_2d(As + s * BMm * BKk, &ma, &full[s], mt * BMm, kb * BKk);
                tma_load_2d(As + s * BMm * BKk + 4096, &ma, &full[s], mt * BMm + 64, kb * BKk);
                tma_load_2d(Bs + s * BNn * BKk, &mb, &full[s], kb * BKk, nt * BNn);
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idesc = idesc_i8<BMm, BNn>() | (1u << 15);  // A MN-major
        for (int kb = 0; kb < nk; ++kb) {
            const int s = kb % ST;
            bar_wait(&full[s], (kb / ST) & 1);
            fence_after_sync();
            if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < 2; ++kk) {
                    const uint64_t da = sdesc_mn_sw64(As + s * BMm * BKk + kk * 2048, 4096);
                    const uint64_t db = sdesc_k_sw64(Bs + s * BNn * BKk) + (uint64_t)(kk * 2);
                    mma_i8(tmem, da, db, idesc, (kb | kk) != 0);
                }
                mma_commit(&empty[s]);
            }
            __syncwarp();
        }
        if (elect_one()) mma_commit(tfull);
        __syncwarp();
    } else {
        bar_wait(tfull, 0);
        fence_after_sync();
        const int q = warp & 3;
        const int row = mt * BMm + q * 32 + lane;
#pragma unroll 1
        for (int c = 0; c < BNn; c += 32) {
            int32_t v[32];
            tmem_ld_32x32b_x32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c, v);
            tmem_ld_wait();
            int32_t* dst = C + (size_t)row * N + nt * BNn + c;
#pragma unroll
            for (int j = 0; j < 32; j += 4) *reinterpret_cast<int4*>(dst + j) = make_int4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        }
    }
    fence_before_sync();
    __syncthreads();
    if (warp == 1) tmem_free<64>(tmem);
}

static PFN_cuTensorMapEncodeTiled_v12000 encode() {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

static CUtensorMap map2d(const int8_t* base, int rows, int K, int box_rows) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)K};
    cuuint32_t box[2] = {BK, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encode()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(base), dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        fprintf(stderr, "tensor map encode failed %d\n", (int)r);
        exit(1);
    }
    return m;
}

template <int BN, int STAGES>
void run(int M, int N, int K, int reps) {
    std::vector<int8_t> hA((size_t)M * K), hB((size_t)N * K);
    std::mt19937 g(1);
    std::uniform_int_distribution<int> d(-64, 64);
    for (auto& x : hA) x = (int8_t)d(g);
    for (auto& x : hB) x = (int8_t)d(g);
    int8_t *A, *B;
    int32_t* C;
    CK(cudaMalloc(&A, hA.size()));
    CK(cudaMalloc(&B, hB.size()));
    CK(cudaMalloc(&C, (size_t)M * N * 4));
    CK(cudaMemcpy(A, hA.data(), hA.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(B, hB.data(), hB.size(), cudaMemcpyHostToDevice));
    CK(cudaMemset(C, 0, (size_t)M * N * 4));
    CUtensorMap ma = map2d(A, M, K, BM), mb = map2d(B, N, K, BN);
    const size_t smem = 1024 + (size_t)STAGES * (BM + BN) * BK + (2 * STAGES + 1) * 8 + 16;
    auto k = i8_gemm_probe<BN, STAGES>;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dim3 grid(M / BM, N / BN);
    k<<<grid, 192, smem>>>(ma, mb, C, M, N, K);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<int32_t> hC((size_t)M * N);
    CK(cudaMemcpy(hC.data(), C, hC.size() * 4, cudaMemcpyDeviceToHost));
    int bad = 0;
    std::mt19937 gs(7);
    for (int t = 0; t < 2000; ++t) {
        const int i = gs() % M, j = gs() % N;
        long long acc = 0;
        for (int kk = 0; kk < K; ++kk) acc += (long long)hA[(size_t)i * K + kk] * hB[(size_t)j * K + kk];
        if (acc != hC[(size_t)i * N + j]) {
            if (bad < 5) fprintf(stderr, "mismatch (%d,%d): got %d want %lld\n", i, j, hC[(size_t)i * N + j], acc);
            ++bad;
        }
    }
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0));
    for (int r = 0; r < reps; ++r) k<<<grid, 192, smem>>>(ma, mb, C, M, N, K);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double ops = 2.0 * M * N * (double)K * reps;
    printf("BN=%d STAGES=%d M=%d N=%d K=%d: %s (%d/2000 bad), %.3f ms/launch, %.1f TOPS\n", BN, STAGES, M, N, K,
           bad ? "FAIL" : "ok", bad, ms / reps, ops / (ms / 1e3) / 1e12);
    cudaFree(A);
    cudaFree(B);
    cudaFree(C);
}

static CUtensorMap map2d_sw64(const int8_t* base, int inner, int outer, int box_inner, int box_outer) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
    cuuint64_t strides[1] = {(cuuint64_t)inner};
    cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encode()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(base), dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        fprintf(stderr, "tensor map encode failed %d\n", (int)r);
        exit(1);
    }
    return m;
}

void run_mn(int M, int N, int K) {
    // A stored [K][M], B stored [N][K]
    std::vector<int8_t> hA((size_t)M * K), hB((size_t)N * K);
    std::mt19937 g(3);
    std::uniform_int_distribution<int> d(-64, 64);
    for (auto& x : hA) x = (int8_t)d(g);
    for (auto& x : hB) x = (int8_t)d(g);
    int8_t *A, *B;
    int32_t* C;
    CK(cudaMalloc(&A, hA.size()));
    CK(cudaMalloc(&B, hB.size()));
    CK(cudaMalloc(&C, (size_t)M * N * 4));
    CK(cudaMemcpy(A, hA.data(), hA.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(B, hB.data(), hB.size(), cudaMemcpyHostToDevice));
    CUtensorMap ma = map2d_sw64(A, M, K, 64, 64), mb = map2d_sw64(B, K, N, 64, 64);
    const size_t smem = 1024 + 4 * (128 + 64) * 64 + 9 * 8 + 16;
    CK(cudaFuncSetAttribute(i8_gemm_mn_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dim3 grid(M / 128, N / 64);
    i8_gemm_mn_probe<<<grid, 192, smem>>>(ma, mb, C, M, N, K);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<int32_t> hC((size_t)M * N);
    CK(cudaMemcpy(hC.data(), C, hC.size() * 4, cudaMemcpyDeviceToHost));
    int bad = 0;
    std::mt19937 gs(9);
    for (int t = 0; t < 2000; ++t) {
        const int i = gs() % M, j = gs() % N;
        long long acc = 0;
        for (int kk = 0; kk < K; ++kk) acc += (long long)hA[(size_t)kk * M + i] * hB[(size_t)j * K + kk];
        if (acc != hC[(size_t)i * N + j]) {
            if (bad < 5) fprintf(stderr, "MN mismatch (%d,%d): got %d want %lld\n", i, j, hC[(size_t)i * N + j], acc);
            ++bad;
        }
    }
    printf("MN-major A: M=%d N=%d K=%d: %s (%d/2000 bad)\n", M, N, K, bad ? "FAIL" : "ok", bad);
    cudaFree(A);
    cudaFree(B);
    cudaFree(C);
}

int main() {
    run_mn(256, 128, 256);
    run_mn(1024, 128, 1024);
    run<128, 4>(1024, 1024, 1024, 5);
    run<256, 4>(4096, 4096, 8192, 20);
    run<128, 6>(4096, 4096, 8192, 20);
    run<256, 4>(8192, 8192, 8192, 10);
    return 0;
}
