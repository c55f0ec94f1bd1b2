// PCIe probe: contiguous pinned copies against the strided row-block copies
// the star-Q host pipeline issues (cudaMemcpy2DAsync, short rows).
// nvcc -O2 -o /tmp/memcpy2d_probe tools/memcpy2d_probe.cu && /tmp/memcpy2d_probe
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

static float time_copy(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height,
                       cudaMemcpyKind kind, cudaStream_t s) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
    float best = 1e30f;
    for (int it = 0; it < 4; ++it) {
        CK(cudaEventRecord(a, s));
        CK(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, kind, s));
        CK(cudaEventRecord(b, s));
        CK(cudaEventSynchronize(b));
        float ms; CK(cudaEventElapsedTime(&ms, a, b));
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    const size_t total = 1ull << 30;  // host tensor, 1 GiB
    char *h, *d;
    CK(cudaMallocHost(&h, total));
    CK(cudaMalloc(&d, total));
    cudaStream_t s; CK(cudaStreamCreate(&s));
    for (size_t i = 0; i < total; i += 4096) h[i] = 1;
    // contiguous 128 MiB
    const size_t blk = 128ull << 20;
    float ms = time_copy(d, blk, h, blk, blk, 1, cudaMemcpyHostToDevice, s);
    printf("H2D contiguous 128 MiB: %.2f ms  %.1f GB/s\n", ms, blk / ms * 1e-6);
    ms = time_copy(h, blk, d, blk, blk, 1, cudaMemcpyDeviceToHost, s);
    printf("D2H contiguous 128 MiB: %.2f ms  %.1f GB/s\n", ms, blk / ms * 1e-6);
    for (size_t width : {512ul, 1024ul, 2048ul, 4096ul, 65536ul, 1048576ul}) {
        const size_t pitch = width * 8, height = blk / width;
        ms = time_copy(d, width, h, pitch, width, height, cudaMemcpyHostToDevice, s);
        printf("H2D 2D rows of %7zu B (pitch x8): %.2f ms  %.1f GB/s\n", width, ms, blk / ms * 1e-6);
        ms = time_copy(h, pitch, d, width, width, height, cudaMemcpyDeviceToHost, s);
        printf("D2H 2D rows of %7zu B (pitch x8): %.2f ms  %.1f GB/s\n", width, ms, blk / ms * 1e-6);
    }
    // both directions at once (two streams), contiguous
    cudaStream_t s2; CK(cudaStreamCreate(&s2));
    char* d2; CK(cudaMalloc(&d2, blk));
    cudaEvent_t a, b, c; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b)); CK(cudaEventCreate(&c));
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(a, s));
    CK(cudaStreamWaitEvent(s2, a, 0));
    for (int i = 0; i < 4; ++i) {
        CK(cudaMemcpyAsync(d, h, blk, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(h + 4 * blk, d2, blk, cudaMemcpyDeviceToHost, s2));
    }
    CK(cudaEventRecord(c, s2));
    CK(cudaStreamWaitEvent(s, c, 0));
    CK(cudaEventRecord(b, s));
    CK(cudaEventSynchronize(b));
    CK(cudaEventElapsedTime(&ms, a, b));
    printf("duplex 4 x 128 MiB each way: %.2f ms  %.1f GB/s per direction\n", ms, 4 * blk / ms * 1e-6);
    // the star-Q host pipeline's shape: 128 MiB row blocks up (1 KB rows, pitch 8 KB)
    // while 256 MiB row blocks come down (1 KB rows, pitch 8 KB)
    {
        char* h2; CK(cudaMallocHost(&h2, 2ull << 30));
        char* d3; CK(cudaMalloc(&d3, 2 * blk));
        const size_t w = 1024, pitch = 8 * w;
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(a, s));
        CK(cudaStreamWaitEvent(s2, a, 0));
        for (int i = 0; i < 8; ++i) {
            CK(cudaMemcpy2DAsync(d, w, h + i * w, pitch, w, blk / w, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpy2DAsync(h2 + i * w, pitch, d3, w, w, 2 * blk / w, cudaMemcpyDeviceToHost, s2));
        }
        CK(cudaEventRecord(c, s2));
        CK(cudaStreamWaitEvent(s, c, 0));
        CK(cudaEventRecord(b, s));
        CK(cudaEventSynchronize(b));
        CK(cudaEventElapsedTime(&ms, a, b));
        printf("pipeline shape: 8 x (128 MiB up + 256 MiB down), strided: %.2f ms  down %.1f GB/s\n", ms,
               16 * blk / ms * 1e-6);
        CK(cudaEventRecord(a, s2));
        for (int i = 0; i < 8; ++i)
            CK(cudaMemcpy2DAsync(h2 + i * w, pitch, d3, w, w, 2 * blk / w, cudaMemcpyDeviceToHost, s2));
        CK(cudaEventRecord(b, s2));
        CK(cudaEventSynchronize(b));
        CK(cudaEventElapsedTime(&ms, a, b));
        printf("down only, 8 x 256 MiB strided: %.2f ms  %.1f GB/s\n", ms, 16 * blk / ms * 1e-6);
        // the 2-D tiled pipeline's downloads: 3-D copies of 128 x 128 x 256 tiles
        // (1 KB runs, 128 per plane, 256 planes) into an 8 KB-pitch, 1024-row slice layout
        char* d4; CK(cudaMalloc(&d4, 32ull << 20));
        for (int rows : {128, 256, 1024}) {
            const size_t tile = (size_t)w * rows * 256;
            const int nt = (int)((1ull << 30) / tile);
            CK(cudaEventRecord(a, s2));
            for (int i = 0; i < nt; ++i) {
                cudaMemcpy3DParms cp = {};
                cp.srcPtr = make_cudaPitchedPtr(d3, w, w, rows);
                cp.dstPtr = make_cudaPitchedPtr(h2 + (i % 8) * w, pitch, pitch, 1024);
                cp.extent = make_cudaExtent(w, rows, 256);
                cp.kind = cudaMemcpyDeviceToHost;
                CK(cudaMemcpy3DAsync(&cp, s2));
            }
            CK(cudaEventRecord(b, s2));
            CK(cudaEventSynchronize(b));
            CK(cudaEventElapsedTime(&ms, a, b));
            printf("down only, 3-D tiles of 1 KB x %d x 256 (%zu MiB each), 1 GiB: %.2f ms  %.1f GB/s\n", rows,
                   tile >> 20, ms, (double)nt * tile / ms * 1e-6);
        }
    }
    return 0;
}
