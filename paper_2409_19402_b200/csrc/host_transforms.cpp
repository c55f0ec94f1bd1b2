// Host-side builders of the structured bases (transforms.cpp:33-95). These
// are tiny n3 x p matrices built once per transform — not part of the hot
// path — so they stay on the host, as in the reference.
#include <cmath>
#include <cstdint>
#include <string>
#include <algorithm>
#include <vector>

#include "internal.h"

using ppc::fail;
using ppc::guarded;

namespace {

// rng.hpp:12-80 (splitmix64 expansion, xoshiro256++, Box-Muller with spare)
struct Xoshiro {
    uint64_t s[4];
    double spare = 0.0;
    bool has_spare = false;
    static uint64_t splitmix(uint64_t& x) {
        x += 0x9e3779b97f4a7c15ULL;
        uint64_t z = x;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    }
    static uint64_t rotl(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }
    explicit Xoshiro(uint64_t seed) {
        uint64_t x = seed;
        for (auto& w : s) w = splitmix(x);
    }
    uint64_t next() {
        const uint64_t r = rotl(s[0] + s[3], 23) + s[0];
        const uint64_t t = s[1] << 17;
        s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3]; s[2] ^= t;
        s[3] = rotl(s[3], 45);
        return r;
    }
    double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    double normal() {
        if (has_spare) {
            has_spare = false;
            return spare;
        }
        double u1 = uniform(), u2 = uniform();
        while (u1 <= 0.0) u1 = uniform();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double th = 2.0 * 3.14159265358979323846 * u2;
        spare = r * std::sin(th);
        has_spare = true;
        return r * std::cos(th);
    }
};

void check_dims(int64_t n3, int64_t p) {
    if (n3 < 1) fail(PPC_ARGUMENT, "transform: n3 must be positive");
    if (p < 1 || p > n3)
        fail(PPC_ARGUMENT, "transform: p=" + std::to_string(p) + " outside [1," + std::to_string(n3) + "]");
}

// singular values of a small dense matrix (one-sided Jacobi), descending
std::vector<double> singular_values(std::vector<double> W, int64_t m, int64_t n) {
    for (int sweep = 0; sweep < 60; ++sweep) {
        bool rot = false;
        for (int64_t i = 0; i < n - 1; ++i)
            for (int64_t j = i + 1; j < n; ++j) {
                double a = 0, b = 0, g = 0;
                for (int64_t r = 0; r < m; ++r) {
                    a += W[r + i * m] * W[r + i * m];
                    b += W[r + j * m] * W[r + j * m];
                    g += W[r + i * m] * W[r + j * m];
                }
                if (g == 0.0 || std::fabs(g) <= 2.220446049250313e-16 * std::sqrt(a * b)) continue;
                rot = true;
                const double z = (b - a) / (2 * g);
                const double t = (z >= 0 ? 1.0 : -1.0) / (std::fabs(z) + std::sqrt(1 + z * z));
                const double c = 1 / std::sqrt(1 + t * t), s = c * t;
                for (int64_t r = 0; r < m; ++r) {
                    const double x = W[r + i * m], y = W[r + j * m];
                    W[r + i * m] = c * x - s * y;
                    W[r + j * m] = s * x + c * y;
                }
            }
        if (!rot) break;
    }
    std::vector<double> s(n);
    for (int64_t j = 0; j < n; ++j) {
        double acc = 0;
        for (int64_t r = 0; r < m; ++r) acc += W[r + j * m] * W[r + j * m];
        s[j] = std::sqrt(acc);
    }
    std::sort(s.begin(), s.end(), [](double x, double y) { return x > y; });
    return s;
}

// matrix_kernels.cpp:48-78: rank gate, Householder QR, first nonnegligible
// entry of each column made positive.
std::vector<double> orthonormalize(const std::vector<double>& A, int64_t n, int64_t p) {
    const auto s = singular_values(A, n, p);
    int64_t rank = 0;
    while (rank < p && s[rank] > 1e-12 * s[0]) ++rank;
    if (rank < p)
        fail(PPC_DEGENERATE, "orthonormalize: input is rank-deficient (rank " + std::to_string(rank) +
                                 " < " + std::to_string(p) + ")");
    std::vector<double> R = A, tau(p, 0.0);
    for (int64_t j = 0; j < p; ++j) {
        double* a = &R[j * n];
        double nrm = 0;
        for (int64_t i = j + 1; i < n; ++i) nrm += a[i] * a[i];
        const double alpha = a[j];
        if (nrm == 0.0) continue;
        const double beta = -std::copysign(std::sqrt(alpha * alpha + nrm), alpha);
        tau[j] = (beta - alpha) / beta;
        const double sc = 1.0 / (alpha - beta);
        for (int64_t i = j + 1; i < n; ++i) a[i] *= sc;
        a[j] = beta;
        for (int64_t c = j + 1; c < p; ++c) {
            double* b = &R[c * n];
            double d = b[j];
            for (int64_t i = j + 1; i < n; ++i) d += a[i] * b[i];
            d *= tau[j];
            b[j] -= d;
            for (int64_t i = j + 1; i < n; ++i) b[i] -= d * a[i];
        }
    }
    std::vector<double> Q(n * p, 0.0);
    for (int64_t j = 0; j < p; ++j) Q[j + j * n] = 1.0;
    for (int64_t j = p - 1; j >= 0; --j) {
        if (tau[j] == 0.0) continue;
        const double* v = &R[j * n];
        for (int64_t c = 0; c < p; ++c) {
            double* b = &Q[c * n];
            double d = b[j];
            for (int64_t i = j + 1; i < n; ++i) d += v[i] * b[i];
            d *= tau[j];
            b[j] -= d;
            for (int64_t i = j + 1; i < n; ++i) b[i] -= d * v[i];
        }
    }
    for (int64_t j = 0; j < p; ++j)
        for (int64_t i = 0; i < n; ++i)
            if (std::fabs(Q[i + j * n]) > 1e-12) {
                if (Q[i + j * n] < 0.0)
                    for (int64_t r = 0; r < n; ++r) Q[r + j * n] = -Q[r + j * n];
                break;
            }
    return Q;
}

}  // namespace

extern "C" {

int ppc_identity_q(int64_t n3, int64_t p, double* Q) {
    return guarded([&] {
        check_dims(n3, p);
        for (int64_t j = 0; j < p; ++j)
            for (int64_t i = 0; i < n3; ++i) Q[i + j * n3] = (i == j) ? 1.0 : 0.0;
    });
}

int ppc_dct_q(int64_t n3, int64_t p, double* Q) {
    return guarded([&] {
        check_dims(n3, p);
        const double n = static_cast<double>(n3);
        for (int64_t j = 0; j < p; ++j) {
            const double w = (j == 0) ? std::sqrt(1.0 / n) : std::sqrt(2.0 / n);
            for (int64_t t = 0; t < n3; ++t)
                Q[t + j * n3] = w * std::cos(3.14159265358979323846 * (2.0 * t + 1.0) * j / (2.0 * n));
        }
    });
}

int ppc_haar_q(int64_t n3, int64_t p, double* Q) {
    return guarded([&] {
        if (n3 != 2 && n3 != 4)
            fail(PPC_ARGUMENT, "haar_transform: n3 must be 2 or 4, got " + std::to_string(n3));
        check_dims(n3, p);
        std::vector<double> H(n3 * n3);
        if (n3 == 2) {
            const double r = 1.0 / std::sqrt(2.0);
            // rows [r r; r -r] (transforms.cpp:49-50), column-major storage
            H = {r, r, r, -r};
        } else {
            const double s = std::sqrt(2.0);
            // rows [1 1 1 1; 1 1 -1 -1; s -s 0 0; 0 0 s -s] * 0.5 (transforms.cpp:52-57)
            const double rows[4][4] = {{1, 1, 1, 1}, {1, 1, -1, -1}, {s, -s, 0, 0}, {0, 0, s, -s}};
            for (int i = 0; i < 4; ++i)
                for (int j = 0; j < 4; ++j) H[i + j * 4] = 0.5 * rows[i][j];
        }
        for (int64_t j = 0; j < p; ++j)
            for (int64_t i = 0; i < n3; ++i) Q[i + j * n3] = H[i + j * n3];
    });
}

int ppc_random_orthogonal_q(int64_t n3, int64_t p, uint64_t seed, double* Q) {
    return guarded([&] {
        check_dims(n3, p);
        Xoshiro rng(seed);
        std::vector<double> G(n3 * n3);
        for (int64_t j = 0; j < n3; ++j)
            for (int64_t i = 0; i < n3; ++i) G[i + j * n3] = rng.normal();  // transforms.cpp:64-66
        const auto F = orthonormalize(G, n3, n3);
        for (int64_t i = 0; i < n3 * p; ++i) Q[i] = F[i];
    });
}

int ppc_orthonormalize(const double* A, int64_t n, int64_t p, double* Q) {
    return guarded([&] {
        if (p < 1 || p > n)
            fail(PPC_ARGUMENT, "orthonormalize: need 1 <= cols <= rows, got " + std::to_string(n) + "x" +
                                   std::to_string(p));
        std::vector<double> a(A, A + n * p);
        for (double x : a)
            if (!std::isfinite(x)) fail(PPC_NUMERIC, "orthonormalize: input has non-finite entries");
        const auto q = orthonormalize(a, n, p);
        for (int64_t i = 0; i < n * p; ++i) Q[i] = q[i];
    });
}

// transforms.cpp:20-27 (+ non-finite check of custom_transform :100-103)
int ppc_check_stiefel(const double* Q, int64_t n3, int64_t p) {
    return guarded([&] {
        check_dims(n3, p);
        for (int64_t i = 0; i < n3 * p; ++i)
            if (!std::isfinite(Q[i])) fail(PPC_NUMERIC, "custom_transform: non-finite entries");
        double res = 0.0;
        for (int64_t a = 0; a < p; ++a)
            for (int64_t b = 0; b < p; ++b) {
                double d = 0.0;
                for (int64_t i = 0; i < n3; ++i) d += Q[i + a * n3] * Q[i + b * n3];
                d -= (a == b) ? 1.0 : 0.0;
                res += d * d;
            }
        res = std::sqrt(res);
        if (!(res <= 1e-10 * static_cast<double>(p)))
            fail(PPC_DEGENERATE, "transform: columns are not orthonormal (residual " +
                                     std::to_string(res) + ")");
    });
}

}  // extern "C"
