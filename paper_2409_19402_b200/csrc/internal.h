// Internal runtime of the ppc engine: per-thread context, error plumbing,
// stream-ordered workspace, launch accounting. Not part of the C-ABI.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <new>
#include <string>

#include "ppc.h"

namespace ppc {

// Typed failure carried from deep inside the engine to the C-ABI boundary,
// where it becomes a status code + ppc_last_error() message.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess)
        fail(PPC_CUDA, std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
                           std::to_string(line) + ")");
}
#define PPC_CUDA_CHECK(x) ::ppc::cuda_check((x), #x, __FILE__, __LINE__)

// Per-thread execution context.
struct Context {
    int device = -1;
    cudaStream_t stream = nullptr;      // user stream (ppc_set_stream) or own
    bool stream_set = false;            // set explicitly (NULL = legacy default stream)
    cudaStream_t own_stream = nullptr;  // created lazily per device
    cudaStream_t copy = nullptr;        // H2D staging stream
    cudaStream_t copy_out = nullptr;    // D2H stream (runs beside the H2D one)
    int* flags[64] = {};                // per-device status words (cudaMalloc'd once)
    int sms = 148;
    int64_t launches = 0;
};
Context& ctx();               // ensures a device is selected (throws PPC_NO_DEVICE)
cudaStream_t stream();        // current stream of this thread
cudaStream_t copy_stream();   // this thread's H2D staging stream (overlap)
cudaStream_t copy_out_stream();  // this thread's D2H stream
// n doubles (n <= 4096, else a plain copy) from device memory to `out`, stream
// ordered on s and synchronized: a one-CTA kernel stores them into mapped pinned
// memory, so the read does not queue on the D2H copy engine behind a bulk
// download in flight on another stream (a pageable cudaMemcpyAsync does).
void read_small(const double* dev, double* out, size_t n, cudaStream_t s);
// This thread's persistent 4-int device status scratch on the current device
// (finiteness flags): allocated once outside the stream-ordered pool, so a
// tiny flag never splits the pool's cached multi-GB blocks.
int* status_words();
inline void count_launch(int n = 1) { ctx().launches += n; }
// Per-device one-time setup (cudaFuncSetAttribute and the like): runs f the
// first time for the current device; `done` holds one bit per device.
template <class F> inline void once_per_device(std::atomic<uint64_t>& done, F&& f) {
    const uint64_t bit = 1ull << (ctx().device & 63);
    if (done.load(std::memory_order_acquire) & bit) return;
    f();
    done.fetch_or(bit, std::memory_order_release);
}
void check_launch(const char* name);  // cudaGetLastError -> PPC_CUDA

// Stream-ordered device buffer (cudaMallocAsync on the current stream; the
// default mempool keeps freed blocks, so steady-state calls do not hit the OS).
// Blocks of >= 256 MB come from an exact-size per-thread cache (runtime.cu).
class DeviceBuffer {
public:
    DeviceBuffer() = default;
    explicit DeviceBuffer(size_t bytes);
    ~DeviceBuffer();
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    DeviceBuffer(DeviceBuffer&& o) noexcept : p_(o.p_), n_(o.n_), dev_(o.dev_) {
        o.p_ = nullptr;
        o.n_ = 0;
        o.dev_ = -1;
    }
    DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
        if (this != &o) {
            release();
            p_ = o.p_;
            n_ = o.n_;
            dev_ = o.dev_;
            o.p_ = nullptr;
            o.n_ = 0;
            o.dev_ = -1;
        }
        return *this;
    }
    void release();
    double* d() const { return static_cast<double*>(p_); }
    template <typename T> T* as() const { return static_cast<T*>(p_); }
    size_t bytes() const { return n_; }
private:
    void* p_ = nullptr;
    size_t n_ = 0;
    int dev_ = -1;  // >= 0: a large block owned by the per-device cache
};
// Frees this thread's cached large blocks on the current device.
void trim_workspace();

// Input/output staging for loc = PPC_HOST: device copies on the current
// stream; for PPC_DEVICE the pointers are passed through untouched.
struct In {
    const double* d = nullptr;
    DeviceBuffer buf;
    In(const double* p, size_t count, int loc);
};
struct Out {
    double* d = nullptr;
    double* host = nullptr;
    size_t count = 0;
    DeviceBuffer buf;
    Out(double* p, size_t count, int loc);
    void finish();  // D2H for host outputs
};

// Optional per-stage device timing (CUDA events on the launching stream),
// enabled by ppc_timing_enable(); used by bench.py for the roofline.
class StageTimer {
public:
    StageTimer(const char* name, cudaStream_t s, double flops = 0.0, double bytes = 0.0);
    ~StageTimer();
    StageTimer(const StageTimer&) = delete;
    StageTimer& operator=(const StageTimer&) = delete;
private:
    const char* name_;
    cudaStream_t s_;
    double flops_, bytes_;
    cudaEvent_t e0_ = nullptr;
};

// Host-side time per named scope (PPC_HOST_PROFILE=1; printed at exit):
// finds the host work that starves the GPU in launch-bound sequences.
class HostProf {
public:
    explicit HostProf(const char* name);
    ~HostProf();
    HostProf(const HostProf&) = delete;
    HostProf& operator=(const HostProf&) = delete;
private:
    const char* name_;
    long long t0_ = -1;
};

void validate_loc(int loc);
void require_positive(int64_t v, const char* what);

void set_error(const std::string& m);
const char* last_error();

// Run a C-ABI body, mapping exceptions to status codes + last_error.
template <class F>
int guarded(F&& f) {
    try {
        f();
        return PPC_OK;
    } catch (const Error& e) {
        set_error(e.what());
        return e.code;
    } catch (const std::bad_alloc&) {
        set_error("host allocation failed");
        return PPC_CUDA;
    } catch (const std::exception& e) {
        set_error(e.what());
        return PPC_CUDA;
    }
}

}  // namespace ppc
