// Per-thread runtime: device/stream selection, error plumbing, stream-ordered
// workspace, host<->device staging. Replaces the reference's L2 runtime
// (parallel.cpp:13-57: slice loops over std::threads) with CUDA grids on one
// device per host thread.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "internal.h"
#include "kernels.cuh"

namespace ppc {

namespace {
thread_local Context t_ctx;
thread_local std::string t_err;
std::once_flag g_pool_once[64];

int visible_devices() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    // PROJPROD_DEVICES caps the count like PROJPROD_THREADS caps workers
    // (parallel.cpp:13-27): unset/invalid = no cap, < 1 clamps to 1.
    const char* env = std::getenv("PROJPROD_DEVICES");
    if (env && *env) {
        char* end = nullptr;
        long cap = std::strtol(env, &end, 10);
        if (end != env) {
            if (cap < 1) cap = 1;
            if (cap < n) n = (int)cap;
        }
    }
    return n;
}

void init_device(int dev) {
    PPC_CUDA_CHECK(cudaSetDevice(dev));
    cudaDeviceProp prop;
    PPC_CUDA_CHECK(cudaGetDeviceProperties(&prop, dev));
    if (prop.major < 10)
        fail(PPC_NO_DEVICE, std::string("device ") + prop.name +
                                " is not sm_100-class; this engine is B200-only");
    t_ctx.device = dev;
    t_ctx.sms = prop.multiProcessorCount;
    if (dev < 64)
        std::call_once(g_pool_once[dev], [dev] {
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
                uint64_t thr = UINT64_MAX;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
            }
        });
}
}  // namespace

Context& ctx() {
    if (t_ctx.device < 0) {
        if (visible_devices() == 0)
            fail(PPC_NO_DEVICE, "no CUDA device visible: the ppc engine has no CPU path");
        init_device(0);
    } else {
        PPC_CUDA_CHECK(cudaSetDevice(t_ctx.device));
    }
    return t_ctx;
}

cudaStream_t stream() {
    Context& c = ctx();
    if (c.stream_set) return c.stream;  // may be the legacy default stream (0)
    if (!c.own_stream) PPC_CUDA_CHECK(cudaStreamCreateWithFlags(&c.own_stream, cudaStreamNonBlocking));
    return c.own_stream;
}

int* status_words() {
    Context& c = ctx();
    const int dev = c.device < 64 ? c.device : 63;
    if (!c.flags[dev]) PPC_CUDA_CHECK(cudaMalloc(&c.flags[dev], 4 * sizeof(int)));
    return c.flags[dev];
}

cudaStream_t copy_out_stream() {
    Context& c = ctx();
    if (!c.copy_out) PPC_CUDA_CHECK(cudaStreamCreateWithFlags(&c.copy_out, cudaStreamNonBlocking));
    return c.copy_out;
}

cudaStream_t copy_stream() {
    Context& c = ctx();
    if (!c.copy) PPC_CUDA_CHECK(cudaStreamCreateWithFlags(&c.copy, cudaStreamNonBlocking));
    return c.copy;
}

namespace {
constexpr size_t kSmallRead = 4096;
__global__ void read_small_kernel(const double* __restrict__ src, double* __restrict__ dst, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}
struct MappedScratch {
    double* h = nullptr;
    ~MappedScratch() {
        if (h) cudaFreeHost(h);
    }
};
thread_local MappedScratch t_scratch;
}  // namespace

void read_small(const double* dev, double* out, size_t n, cudaStream_t s) {
    if (n == 0) return;
    if (n > kSmallRead) {
        PPC_CUDA_CHECK(cudaMemcpyAsync(out, dev, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
        PPC_CUDA_CHECK(cudaStreamSynchronize(s));
        return;
    }
    if (!t_scratch.h)
        PPC_CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&t_scratch.h), sizeof(double) * kSmallRead,
                                     cudaHostAllocMapped | cudaHostAllocPortable));
    double* dptr = nullptr;
    PPC_CUDA_CHECK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dptr), t_scratch.h, 0));
    read_small_kernel<<<1, 256, 0, s>>>(dev, dptr, (int)n);
    count_launch();
    check_launch("read_small");
    PPC_CUDA_CHECK(cudaStreamSynchronize(s));
    std::copy(t_scratch.h, t_scratch.h + n, out);
}

void check_launch(const char* name) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) fail(PPC_CUDA, std::string(name) + " launch: " + cudaGetErrorString(e));
}

// Large buffers (>= 32 MB: tensor-sized transforms, digit planes, slice
// Grams) recur with identical sizes from call to call. They are kept in a
// per-thread, per-device exact-size cache instead of going back to the
// stream-ordered pool: freed multi-GB blocks that the pool later carves small
// allocations from made the next call map fresh memory, measured as 10..400 ms
// stalls inside the Gram. A cached block carries the event of its release, so
// reuse on another stream still waits for the last user.
namespace {
constexpr size_t kBigBytes = size_t(32) << 20;
struct BigBlock {
    size_t bytes;
    void* p;
    cudaEvent_t done;
};
struct BigCache {
    std::vector<BigBlock> free;
    size_t held = 0;
};
thread_local BigCache t_big[64];

size_t big_cap(int dev) {  // keep at most half of the device memory cached
    static size_t cap[64] = {};
    if (!cap[dev]) {
        size_t fr = 0, tot = 0;
        cap[dev] = cudaMemGetInfo(&fr, &tot) == cudaSuccess ? tot / 2 : (size_t(64) << 30);
    }
    return cap[dev];
}

void big_drop(BigCache& c, size_t i) {
    cudaEventSynchronize(c.free[i].done);
    cudaEventDestroy(c.free[i].done);
    cudaFree(c.free[i].p);
    c.held -= c.free[i].bytes;
    c.free.erase(c.free.begin() + (long)i);
}
}  // namespace

// The pool keeps freed memory (release threshold: unlimited); under memory
// pressure it is returned to the driver once the stream's frees are done.
void release_pool_reserve(cudaStream_t s) {
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        cudaStreamSynchronize(s);
        cudaMemPoolTrimTo(pool, 0);
    }
    cudaGetLastError();
}

void trim_workspace() {
    Context& c = ctx();
    BigCache& bc = t_big[c.device < 64 ? c.device : 63];
    while (!bc.free.empty()) big_drop(bc, bc.free.size() - 1);
}

DeviceBuffer::DeviceBuffer(size_t bytes) : n_(bytes) {
    HostProf hp_("DeviceBuffer");
    if (!bytes) return;
    cudaStream_t s = stream();
    if (bytes >= kBigBytes) {
        const int dev = ctx().device < 64 ? ctx().device : 63;
        dev_ = dev;
        BigCache& c = t_big[dev];
        for (size_t i = 0; i < c.free.size(); ++i)
            if (c.free[i].bytes == bytes) {
                p_ = c.free[i].p;
                PPC_CUDA_CHECK(cudaStreamWaitEvent(s, c.free[i].done, 0));
                PPC_CUDA_CHECK(cudaEventDestroy(c.free[i].done));
                c.held -= bytes;
                c.free.erase(c.free.begin() + (long)i);
                return;
            }
        // not cached: a plain allocation (outside the pool) of this size
        static const bool trace = std::getenv("PPC_TRACE_ALLOC") != nullptr;
        if (trace)
            fprintf(stderr, "[alloc] miss %.3f GB (cache holds %zu blocks, %.1f GB)\n", bytes / 1e9, c.free.size(),
                    c.held / 1e9);
        cudaError_t e = cudaMalloc(&p_, bytes);
        while (e == cudaErrorMemoryAllocation && !c.free.empty()) {  // make room from the cache
            cudaGetLastError();
            big_drop(c, 0);
            e = cudaMalloc(&p_, bytes);
        }
        if (e == cudaErrorMemoryAllocation) {  // and from the stream-ordered pool's reserve
            cudaGetLastError();
            release_pool_reserve(s);
            e = cudaMalloc(&p_, bytes);
        }
        PPC_CUDA_CHECK(e);
        return;
    }
    static const bool trace = std::getenv("PPC_TRACE_ALLOC") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    cudaError_t e = cudaMallocAsync(&p_, bytes, s);
    if (e == cudaErrorMemoryAllocation) {
        // memory pressure (another allocator, or a caller's own buffers): the
        // workspace cache gives its blocks back, then the allocation retries
        cudaGetLastError();
        trim_workspace();
        release_pool_reserve(s);
        e = cudaMallocAsync(&p_, bytes, s);
    }
    PPC_CUDA_CHECK(e);
    if (trace) {
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        if (ms > 2.0) fprintf(stderr, "[alloc] pool %.1f MB took %.1f ms\n", bytes / 1e6, ms);
    }
}
DeviceBuffer::~DeviceBuffer() { release(); }
void DeviceBuffer::release() {
    HostProf hp_("DeviceBuffer::release");
    if (p_) {
        if (dev_ >= 0) {
            BigCache& c = t_big[dev_];
            cudaEvent_t ev = nullptr;
            if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess &&
                cudaEventRecord(ev, stream()) == cudaSuccess) {
                c.free.push_back({n_, p_, ev});
                c.held += n_;
                while (c.held > big_cap(dev_) && c.free.size() > 1) {  // oldest first
                    if (std::getenv("PPC_TRACE_ALLOC"))
                        fprintf(stderr, "[alloc] drop %.3f GB over the cap\n", c.free[0].bytes / 1e9);
                    big_drop(c, 0);
                }
            } else {
                if (ev) cudaEventDestroy(ev);
                cudaDeviceSynchronize();
                cudaFree(p_);
            }
        } else {
            cudaFreeAsync(p_, stream());
        }
    }
    p_ = nullptr;
    n_ = 0;
    dev_ = -1;
}

void validate_loc(int loc) {
    if (loc != PPC_HOST && loc != PPC_DEVICE) fail(PPC_ARGUMENT, "loc must be PPC_HOST or PPC_DEVICE");
}

void require_positive(int64_t v, const char* what) {
    if (v < 1) fail(PPC_SHAPE, std::string(what) + " must be positive");
}

In::In(const double* p, size_t count, int loc) {
    if (loc == PPC_DEVICE || count == 0) {
        d = p;
        return;
    }
    if (!p) fail(PPC_ARGUMENT, "null input pointer");
    buf = DeviceBuffer(count * sizeof(double));
    PPC_CUDA_CHECK(cudaMemcpyAsync(buf.d(), p, count * sizeof(double), cudaMemcpyHostToDevice, stream()));
    d = buf.d();
}

Out::Out(double* p, size_t n, int loc) : count(n) {
    if (loc == PPC_DEVICE || n == 0) {
        d = p;
        return;
    }
    if (!p) fail(PPC_ARGUMENT, "null output pointer");
    host = p;
    buf = DeviceBuffer(n * sizeof(double));
    d = buf.d();
}

void Out::finish() {
    if (host)
        PPC_CUDA_CHECK(cudaMemcpyAsync(host, d, count * sizeof(double), cudaMemcpyDeviceToHost, stream()));
}

// ---------------------------------------------------------- stage timing
namespace {
struct StageRec {
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
    double flops = 0.0, bytes = 0.0;
    int64_t launches = 0;
};
thread_local bool t_timing = false;
thread_local std::map<std::string, StageRec> t_stages;
}  // namespace

StageTimer::StageTimer(const char* name, cudaStream_t s, double flops, double bytes)
    : name_(name), s_(s), flops_(flops), bytes_(bytes) {
    HostProf hp_("StageTimer");
    if (!t_timing) return;
    cudaEventCreate(&e0_);
    cudaEventRecord(e0_, s_);
}
StageTimer::~StageTimer() {
    if (!e0_) return;
    cudaEvent_t e1;
    cudaEventCreate(&e1);
    cudaEventRecord(e1, s_);
    StageRec& r = t_stages[name_];
    r.ev.emplace_back(e0_, e1);
    r.flops += flops_;
    r.bytes += bytes_;
    r.launches += 1;
}

namespace {
struct HostProfTable {
    std::map<std::string, std::pair<double, long long>> t;  // ms, calls
    ~HostProfTable() {
        if (t.empty()) return;
        std::vector<std::pair<double, std::string>> v;
        for (auto& kv : t) v.push_back({kv.second.first, kv.first});
        std::sort(v.rbegin(), v.rend());
        for (auto& e : v)
            fprintf(stderr, "[host] %-28s %9.3f ms  %7lld calls  %8.2f us/call\n", e.second.c_str(), e.first,
                    t[e.second].second, 1e3 * e.first / (double)t[e.second].second);
    }
};
HostProfTable g_hostprof;
std::mutex g_hostprof_mu;
bool host_prof_on() {
    static const bool on = std::getenv("PPC_HOST_PROFILE") != nullptr;
    return on;
}
long long now_ns() {
    return std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch())
        .count();
}
}  // namespace

HostProf::HostProf(const char* name) : name_(name) {
    if (host_prof_on()) t0_ = now_ns();
}
HostProf::~HostProf() {
    if (t0_ < 0) return;
    const double ms = (now_ns() - t0_) / 1e6;
    std::lock_guard<std::mutex> g(g_hostprof_mu);
    auto& e = g_hostprof.t[name_];
    e.first += ms;
    e.second += 1;
}

void set_error(const std::string& m) { t_err = m; }
const char* last_error() { return t_err.c_str(); }

}  // namespace ppc

extern "C" {

const char* ppc_last_error(void) { return ppc::last_error(); }
int ppc_version(void) { return PPC_VERSION; }

int ppc_device_count(void) { return ppc::visible_devices(); }

int ppc_set_device(int device) {
    try {
        int n = ppc::visible_devices();
        if (device < 0 || device >= n) ppc::fail(PPC_ARGUMENT, "ppc_set_device: no such device");
        if (ppc::t_ctx.device != device) {
            ppc::t_ctx.stream = nullptr;
            ppc::t_ctx.stream_set = false;
            ppc::t_ctx.own_stream = nullptr;
            ppc::t_ctx.copy = nullptr;
        }
        ppc::init_device(device);
        return 0;
    } catch (const ppc::Error& e) {
        ppc::set_error(e.what());
        return e.code;
    }
}

int ppc_set_stream(void* s) {
    try {
        ppc::ctx().stream = static_cast<cudaStream_t>(s);
        ppc::ctx().stream_set = true;
        return 0;
    } catch (const ppc::Error& e) {
        ppc::set_error(e.what());
        return e.code;
    }
}

void* ppc_get_stream(void) {
    try {
        return ppc::stream();
    } catch (...) {
        return nullptr;
    }
}

int ppc_synchronize(void) {
    try {
        PPC_CUDA_CHECK(cudaStreamSynchronize(ppc::stream()));
        return 0;
    } catch (const ppc::Error& e) {
        ppc::set_error(e.what());
        return e.code;
    }
}

int ppc_trim_workspace(void) {
    try {
        ppc::trim_workspace();
        return 0;
    } catch (const ppc::Error& e) {
        ppc::set_error(e.what());
        return e.code;
    }
}

int ppc_timing_enable(int on) {
    ppc::t_timing = on != 0;
    return 0;
}

// JSON object {"stage": {"ms": total, "n": launches, "flops": F, "bytes": B}, ...}
// of everything recorded since the last reset; synchronizes the events.
int ppc_timing_report(char* buf, int64_t cap, int reset) {
    return ppc::guarded([&] {
        std::string out = "{";
        bool first = true;
        for (auto& kv : ppc::t_stages) {
            double ms = 0.0;
            for (auto& pr : kv.second.ev) {
                PPC_CUDA_CHECK(cudaEventSynchronize(pr.second));
                float t = 0.f;
                PPC_CUDA_CHECK(cudaEventElapsedTime(&t, pr.first, pr.second));
                ms += t;
            }
            char tmp[256];
            snprintf(tmp, sizeof tmp, "%s\"%s\": {\"ms\": %.6f, \"n\": %lld, \"flops\": %.6e, \"bytes\": %.6e}",
                     first ? "" : ", ", kv.first.c_str(), ms, (long long)kv.second.launches,
                     kv.second.flops, kv.second.bytes);
            out += tmp;
            first = false;
        }
        out += "}";
        if ((int64_t)out.size() + 1 > cap) ppc::fail(PPC_ARGUMENT, "timing report buffer too small");
        memcpy(buf, out.c_str(), out.size() + 1);
        if (reset) {
            for (auto& kv : ppc::t_stages)
                for (auto& pr : kv.second.ev) {
                    cudaEventDestroy(pr.first);
                    cudaEventDestroy(pr.second);
                }
            ppc::t_stages.clear();
        }
    });
}

int64_t ppc_launch_count(int reset) {
    int64_t n = ppc::t_ctx.launches;
    if (reset) ppc::t_ctx.launches = 0;
    return n;
}

}  // extern "C"
