// PT3 container I/O (io.cpp:52-112, io.hpp:11-22) straight into the engine's
// layout. The payload is already mode-1 fastest, i.e. the device tensor
// layout, so a file streams into (or out of) device memory in large chunks.
// Two pinned staging buffers alternate: the disk read of chunk i+1 runs
// while chunk i is in flight over PCIe on the copy stream (and the reverse
// for writes). Host-pointer calls never touch CUDA.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cstdlib>
#include <cstring>
#include <string>

#include "internal.h"

namespace ppc {
namespace {

constexpr size_t kHeader = 36;
constexpr uint32_t kVersion = 1;  // kPt3Version (io.hpp:23)

void put_u32(unsigned char* at, uint32_t v) {
    for (int i = 0; i < 4; ++i) at[i] = (unsigned char)(v >> (8 * i));
}
void put_u64(unsigned char* at, uint64_t v) {
    for (int i = 0; i < 8; ++i) at[i] = (unsigned char)(v >> (8 * i));
}
uint32_t get_u32(const unsigned char* at) {
    uint32_t v = 0;
    for (int i = 0; i < 4; ++i) v |= (uint32_t)at[i] << (8 * i);
    return v;
}
uint64_t get_u64(const unsigned char* at) {
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= (uint64_t)at[i] << (8 * i);
    return v;
}

[[noreturn]] void bad(const char* path, const std::string& why) {
    fail(PPC_FORMAT, std::string(path) + ": " + why);
}

struct Fd {
    int fd = -1;
    ~Fd() {
        if (fd >= 0) ::close(fd);
    }
};

// io.cpp:72-101: header checks in the reference's order, then the exact
// payload size. Returns the element count.
uint64_t read_header(const char* path, int fd, int64_t* n1, int64_t* n2, int64_t* n3) {
    unsigned char h[kHeader];
    ssize_t got = ::pread(fd, h, kHeader, 0);
    if (got != (ssize_t)kHeader) bad(path, "truncated header");
    if (std::memcmp(h, "PT3\0", 4) != 0) bad(path, "bad magic");
    const uint32_t version = get_u32(h + 4);
    if (version != kVersion) bad(path, "unsupported version " + std::to_string(version));
    if (h[8] != 1) bad(path, "unsupported dtype " + std::to_string((int)h[8]));
    if (h[9] != 0) bad(path, "unsupported field flags " + std::to_string((int)h[9]));
    const uint64_t a = get_u64(h + 12), b = get_u64(h + 20), c = get_u64(h + 28);
    if (a == 0 || b == 0 || c == 0) bad(path, "zero extent");
    constexpr uint64_t kMaxElems = uint64_t{1} << 59;
    if (a > kMaxElems / b || (a * b) > kMaxElems / c)
        bad(path, "element count overflows the addressable payload");
    const uint64_t elems = a * b * c;
    struct stat st;
    if (::fstat(fd, &st) != 0) bad(path, "cannot stat");
    if ((uint64_t)st.st_size != kHeader + elems * sizeof(double))
        bad(path, "payload size mismatch (truncated or trailing bytes)");
    *n1 = (int64_t)a;
    *n2 = (int64_t)b;
    *n3 = (int64_t)c;
    return elems;
}

int open_read(const char* path) {
    if (!path) fail(PPC_ARGUMENT, "pt3: null path");
    const int fd = ::open(path, O_RDONLY | O_CLOEXEC);
    if (fd < 0) bad(path, "cannot open");
    return fd;
}

size_t staging_bytes() {
    static const size_t v = [] {
        const char* e = std::getenv("PPC_PT3_CHUNK_KB");
        const long kb = e ? std::atol(e) : 64 * 1024;
        return (size_t)std::max(4L, kb) * 1024;
    }();
    return v;
}

void pread_all(const char* path, int fd, void* dst, size_t n, uint64_t off) {
    char* p = static_cast<char*>(dst);
    while (n) {
        const ssize_t r = ::pread(fd, p, n, (off_t)off);
        if (r < 0 && errno == EINTR) continue;
        if (r <= 0) bad(path, "short read");
        p += r;
        n -= (size_t)r;
        off += (uint64_t)r;
    }
}

void pwrite_all(const char* path, int fd, const void* src, size_t n, uint64_t off) {
    const char* p = static_cast<const char*>(src);
    while (n) {
        const ssize_t r = ::pwrite(fd, p, n, (off_t)off);
        if (r < 0 && errno == EINTR) continue;
        if (r <= 0) bad(path, "short write");
        p += r;
        n -= (size_t)r;
        off += (uint64_t)r;
    }
}

// Two pinned staging buffers with completion events on the copy stream.
struct Staging {
    void* buf[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    size_t bytes;
    explicit Staging(size_t b) : bytes(b) {
        for (int i = 0; i < 2; ++i) {
            PPC_CUDA_CHECK(cudaHostAlloc(&buf[i], bytes, cudaHostAllocDefault));
            PPC_CUDA_CHECK(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
        }
    }
    ~Staging() {
        for (int i = 0; i < 2; ++i) {
            if (ev[i]) cudaEventDestroy(ev[i]);
            if (buf[i]) cudaFreeHost(buf[i]);
        }
    }
};

}  // namespace
}  // namespace ppc

using namespace ppc;

extern "C" {

int ppc_pt3_info(const char* path, int64_t* n1, int64_t* n2, int64_t* n3) {
    return guarded([&] {
        if (!n1 || !n2 || !n3) fail(PPC_ARGUMENT, "pt3_info: null output");
        Fd f{open_read(path)};
        read_header(path, f.fd, n1, n2, n3);
    });
}

int ppc_pt3_read(const char* path, double* dst, int64_t count, int loc) {
    return guarded([&] {
        validate_loc(loc);
        Fd f{open_read(path)};
        int64_t a, b, c;
        const uint64_t elems = read_header(path, f.fd, &a, &b, &c);
        if (count < 0 || (uint64_t)count != elems)
            fail(PPC_SHAPE, std::string(path) + ": holds " + std::to_string(elems) +
                                " elements, destination has " + std::to_string(count));
        if (!dst) fail(PPC_ARGUMENT, "pt3_read: null destination");
        const size_t total = (size_t)elems * sizeof(double);
        if (loc == PPC_HOST) {
            pread_all(path, f.fd, dst, total, kHeader);
            return;
        }
        PPC_CUDA_CHECK(cudaStreamSynchronize(stream()));  // earlier users of dst are done
        cudaStream_t cs = copy_stream();
        Staging st(std::min(staging_bytes(), total));
        char* d = reinterpret_cast<char*>(dst);
        size_t done = 0;
        for (int i = 0; done < total; i ^= 1) {
            const size_t n = std::min(st.bytes, total - done);
            PPC_CUDA_CHECK(cudaEventSynchronize(st.ev[i]));  // buffer i free again
            pread_all(path, f.fd, st.buf[i], n, kHeader + done);
            PPC_CUDA_CHECK(cudaMemcpyAsync(d + done, st.buf[i], n, cudaMemcpyHostToDevice, cs));
            PPC_CUDA_CHECK(cudaEventRecord(st.ev[i], cs));
            done += n;
        }
        // the tensor is complete for work queued on the engine stream
        PPC_CUDA_CHECK(cudaStreamSynchronize(cs));
    });
}

int ppc_pt3_write(const char* path, const double* src, int64_t n1, int64_t n2, int64_t n3, int loc) {
    return guarded([&] {
        validate_loc(loc);
        if (!path) fail(PPC_ARGUMENT, "pt3: null path");
        require_positive(n1, "n1");
        require_positive(n2, "n2");
        require_positive(n3, "n3");
        if (!src) fail(PPC_ARGUMENT, "pt3_write: null source");
        unsigned char h[kHeader] = {};
        std::memcpy(h, "PT3\0", 4);
        put_u32(h + 4, kVersion);
        h[8] = 1;  // float64
        h[9] = 0;  // field flags
        put_u64(h + 12, (uint64_t)n1);
        put_u64(h + 20, (uint64_t)n2);
        put_u64(h + 28, (uint64_t)n3);
        Fd f;
        f.fd = ::open(path, O_WRONLY | O_CREAT | O_TRUNC | O_CLOEXEC, 0644);
        if (f.fd < 0) fail(PPC_FORMAT, std::string(path) + ": cannot open for writing");
        pwrite_all(path, f.fd, h, kHeader, 0);
        const size_t total = (size_t)n1 * n2 * n3 * sizeof(double);
        if (loc == PPC_HOST) {
            pwrite_all(path, f.fd, src, total, kHeader);
            return;
        }
        // everything queued on the engine stream (the producer) first
        PPC_CUDA_CHECK(cudaStreamSynchronize(stream()));
        cudaStream_t cs = copy_stream();
        Staging st(std::min(staging_bytes(), total));
        const char* s = reinterpret_cast<const char*>(src);
        size_t issued = 0, written = 0;
        size_t len[2] = {0, 0};
        // prime: D2H of chunk 0, then keep one chunk in flight while writing
        len[0] = std::min(st.bytes, total);
        PPC_CUDA_CHECK(cudaMemcpyAsync(st.buf[0], s, len[0], cudaMemcpyDeviceToHost, cs));
        PPC_CUDA_CHECK(cudaEventRecord(st.ev[0], cs));
        issued = len[0];
        for (int i = 0; written < total; i ^= 1) {
            if (issued < total) {
                const int j = i ^ 1;
                len[j] = std::min(st.bytes, total - issued);
                PPC_CUDA_CHECK(cudaMemcpyAsync(st.buf[j], s + issued, len[j], cudaMemcpyDeviceToHost, cs));
                PPC_CUDA_CHECK(cudaEventRecord(st.ev[j], cs));
                issued += len[j];
            }
            PPC_CUDA_CHECK(cudaEventSynchronize(st.ev[i]));
            pwrite_all(path, f.fd, st.buf[i], len[i], kHeader + written);
            written += len[i];
        }
    });
}

}  // extern "C"
