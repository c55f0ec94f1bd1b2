// C++ API drop-in test: the reference's own test cases (proj/tests/*.cpp,
// restated without doctest/Eigen) run against libprojprod.so -> libppc.so.
// Exit code 0 = all passed. Needs a B200.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

#include <unistd.h>

#include "projprod/decompositions.hpp"
#include "projprod/errors.hpp"
#include "projprod/io.hpp"
#include "projprod/metrics.hpp"
#include "projprod/parallel.hpp"
#include "projprod/star_products.hpp"

using namespace projprod;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                                   \
    do {                                                                           \
        ++g_checks;                                                                \
        if (!(c)) {                                                                \
            ++g_fail;                                                              \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);      \
        }                                                                          \
    } while (0)
template <class E, class F>
static void check_throws(F f, const char* what) {
    ++g_checks;
    try {
        f();
    } catch (const E&) {
        return;
    } catch (...) {
    }
    ++g_fail;
    std::fprintf(stderr, "FAIL: expected exception: %s\n", what);
}

static Tensor3 make_tube(std::vector<double> v) {
    Tensor3 t(1, 1, (Index)v.size());
    for (Index k = 0; k < t.n3(); ++k) t(0, 0, k) = v[(size_t)k];
    return t;
}
static Tensor3 counterexample() {  // tests/support/common.hpp:15-22
    Tensor3 A(2, 2, 2);
    A(0, 0, 0) = 1; A(1, 1, 0) = 1; A(0, 0, 1) = 1; A(1, 1, 1) = -1;
    return A;
}
static Tensor3 seeded(Index n1, Index n2, Index n3, unsigned s) {
    Tensor3 A(n1, n2, n3);
    unsigned x = s * 2654435761u + 1;
    for (Index i = 0; i < A.size(); ++i) {
        x = x * 1664525u + 1013904223u;
        A.data()[i] = ((x >> 8) * (1.0 / 16777216.0)) - 0.5;
    }
    return A;
}

int main() {
    const double s2 = std::sqrt(2.0);
    // test_star_products.cpp:70-78 — worked projected products
    {
        Tensor3 a = make_tube({2, 4, 6, 8}), b = make_tube({1, -1, 1, 0});
        StarContext ctx(haar_transform(4, 2));
        Tensor3 ab = star_q_product(a, b, ctx);
        const double w[4] = {3, 3, 3, 0};
        for (int k = 0; k < 4; ++k) CHECK(std::fabs(ab(0, 0, k) - w[k]) <= 1e-12);
        Matrix H4 = haar_transform(4, 4).Q;
        StarContext perp(custom_transform(H4.rightCols(2)));
        Tensor3 c = star_q_product(a, b, perp);
        const double w2[4] = {-1, 1, 0, 8};
        for (int k = 0; k < 4; ++k) CHECK(std::fabs(c(0, 0, k) - w2[k]) <= 1e-12);
        // identity acts as projection: [3,3,6,0]
        Tensor3 ia = star_q_product(star_q_identity(1, ctx), a, ctx);
        const double w3[4] = {3, 3, 6, 0};
        for (int k = 0; k < 4; ++k) CHECK(std::fabs(ia(0, 0, k) - w3[k]) <= 1e-12);
    }
    // test_tensor.cpp:101-121 — mode-3 product KAT
    {
        Tensor3 a = make_tube({2, 4, 6, 8});
        Matrix Q = haar_transform(4, 2).Q;
        Tensor3 ah = mode3_product(a, Q.transpose());
        CHECK(std::fabs(ah(0, 0, 0) - (3 + 3 * s2)) <= 1e-14 * (3 + 3 * s2));
        CHECK(std::fabs(ah(0, 0, 1) - (3 - 3 * s2)) <= 1e-13);
        check_throws<shape_error>([&] { mode3_product(a, Matrix::Identity(3, 3)); }, "mode3 shape");
    }
    // test_tensor.cpp:87-99 — general mode unfold (host-side layout)
    {
        Tensor3 A = counterexample();
        Matrix u3 = mode_unfold(A, 3), w3 = mode3_unfold(A);
        bool same = u3.rows() == w3.rows() && u3.cols() == w3.cols();
        for (Index i = 0; same && i < u3.size(); ++i) same = u3.data()[i] == w3.data()[i];
        CHECK(same);
        Tensor3 I2(2, 2, 2);
        I2(0, 0, 0) = I2(1, 1, 0) = I2(0, 0, 1) = I2(1, 1, 1) = 1.0;
        const double w1[2][4] = {{1, 0, 1, 0}, {0, 1, 0, 1}};
        Matrix u1 = mode_unfold(I2, 1);
        CHECK(u1.rows() == 2 && u1.cols() == 4);
        for (Index r = 0; r < 2; ++r)
            for (Index c = 0; c < 4; ++c) CHECK(u1(r, c) == w1[r][c]);
        Matrix u2 = mode_unfold(Tensor3(3, 2, 2), 2);
        CHECK(u2.rows() == 2 && u2.cols() == 6);
        for (Index i = 0; i < u2.size(); ++i) CHECK(u2.data()[i] == 0.0);
        // mode 2 column order i + k n1
        Tensor3 S = seeded(3, 4, 2, 11);
        Matrix s2u = mode_unfold(S, 2);
        for (Index k = 0; k < 2; ++k)
            for (Index i = 0; i < 3; ++i)
                for (Index j = 0; j < 4; ++j) CHECK(s2u(j, i + k * 3) == S(i, j, k));
        check_throws<argument_error>([&] { mode_unfold(A, 4); }, "mode_unfold mode");
    }
    // test_tensor.cpp:123-134 — mode products against index loops (3 x 4 x 5, M 6 x ext)
    {
        Tensor3 A = seeded(3, 4, 5, 7);
        for (int mode = 1; mode <= 3; ++mode) {
            const Index ext = mode == 1 ? 3 : (mode == 2 ? 4 : 5);
            Tensor3 Ms = seeded(6, ext, 1, 20 + (unsigned)mode);
            Matrix M(6, ext);
            for (Index r = 0; r < 6; ++r)
                for (Index c = 0; c < ext; ++c) M(r, c) = Ms(r, c, 0);
            Tensor3 got = mode_product(A, M, mode);
            double err2 = 0.0, ref2 = 0.0;
            const Index o1 = mode == 1 ? 6 : 3, o2 = mode == 2 ? 6 : 4, o3 = mode == 3 ? 6 : 5;
            CHECK(got.n1() == o1 && got.n2() == o2 && got.n3() == o3);
            for (Index i = 0; i < o1; ++i)
                for (Index j = 0; j < o2; ++j)
                    for (Index k = 0; k < o3; ++k) {
                        double w = 0.0;
                        for (Index t = 0; t < ext; ++t)
                            w += mode == 1 ? M(i, t) * A(t, j, k) : (mode == 2 ? M(j, t) * A(i, t, k) : M(k, t) * A(i, j, t));
                        err2 += (got(i, j, k) - w) * (got(i, j, k) - w);
                        ref2 += w * w;
                    }
            CHECK(std::sqrt(err2) <= 1e-13 * std::max(1.0, std::sqrt(ref2)));
        }
        check_throws<shape_error>([&] { mode_product(A, Matrix::Identity(4, 4), 1); }, "mode_product(1) shape");
        check_throws<shape_error>([&] { mode_product(A, Matrix::Identity(3, 3), 2); }, "mode_product(2) shape");
        check_throws<argument_error>([&] { mode_product(A, Matrix::Identity(3, 3), 0); }, "mode_product mode");
    }
    // parallel.cpp:13-57 — worker cap, coverage of [0, n), first exception rethrown
    {
        CHECK(max_threads() >= 1);
        setenv("PROJPROD_THREADS", "3", 1);
        CHECK(max_threads() <= 3);
        setenv("PROJPROD_THREADS", "-5", 1);
        CHECK(max_threads() == 1);
        setenv("PROJPROD_THREADS", "junk", 1);
        CHECK(max_threads() >= 1);
        setenv("PROJPROD_THREADS", "4", 1);
        std::vector<int> hit(1000, 0);
        parallel_for(1000, [&](std::ptrdiff_t i) { hit[(size_t)i] += 1; });
        bool once = true;
        for (int h : hit) once = once && h == 1;
        CHECK(once);
        parallel_for(0, [&](std::ptrdiff_t) { CHECK(false); });
        check_throws<argument_error>(
            [&] { parallel_for(64, [&](std::ptrdiff_t i) { if (i == 37) throw argument_error("boom"); }); },
            "parallel_for rethrow");
        unsetenv("PROJPROD_THREADS");
    }
    // test_tensor.cpp:144-149 — facewise tube
    {
        Tensor3 ab = facewise_product(make_tube({1, 2, 3}), make_tube({4, 5, -6}));
        CHECK(ab(0, 0, 0) == 4.0 && ab(0, 0, 1) == 10.0 && ab(0, 0, 2) == -18.0);
        check_throws<shape_error>([&] { facewise_product(counterexample(), Tensor3(3, 2, 2)); }, "facewise");
    }
    // test_tensor.cpp:160-165 — Frobenius norm
    CHECK(std::fabs(frobenius_norm(counterexample()) - 2.0) <= 1e-15 * 2);
    CHECK(frobenius_norm(Tensor3(3, 3, 3)) == 0.0);
    // test_decompositions.cpp:61-78 — error splits
    {
        Tensor3 A = counterexample();
        Transform Tdd = data_dependent_transform(A, 1);
        ApproxError e1 = tsvdq_error(A, tsvdq(A, Tdd, 1));
        CHECK(std::fabs(e1.total - std::sqrt(3.0)) <= 1e-12);
        CHECK(std::fabs(e1.eckart_young - 1.0) <= 1e-12);
        CHECK(std::fabs(e1.projection - s2) <= 1e-12);
        Transform Th = haar_transform(2, 1);
        TsvdqFactors F = tsvdq(A, Th, 1);
        ApproxError e2 = tsvdq_error(A, F);
        CHECK(std::fabs(e2.total - s2) <= 1e-12);
        CHECK(std::fabs(e2.eckart_young) <= 1e-12);
        CHECK(std::fabs(e2.projection - s2) <= 1e-12);
        // test_metrics.cpp:19-24
        CHECK(std::fabs(relative_error(A, tsvdq_reconstruct(F)) - s2 / 2) <= 1e-12);
        CHECK(std::fabs(tsvdq_relative_error(A, F) - s2 / 2) <= 1e-12);
        check_throws<degenerate_input_error>([&] { relative_error(Tensor3(2, 2, 2), A); }, "zero ref");
    }
    // test_transforms.cpp:112-121 — projection error
    CHECK(std::fabs(projection_error(make_tube({2, 4, 6, 8}), haar_transform(4, 2)) - std::sqrt(66.0)) <= 1e-12);
    // test_decompositions.cpp:27-59 — factor contracts and sigma-form reconstruction
    {
        Tensor3 A = seeded(5, 4, 6, 41);
        Transform T = dct_transform(6, 3);
        TsvdqFactors F = tsvdq(A, T, 3);
        CHECK(F.Uhat.size() == 3 && F.Vhat.size() == 3);
        for (size_t i = 0; i < 3; ++i) {
            const Matrix& U = F.Uhat[i];
            CHECK((U.transpose() * U - Matrix::Identity(3, 3)).norm() <= 1e-10 * 3);
            const Vector& s = F.shat[i];
            for (Index j = 0; j + 1 < s.size(); ++j) CHECK(s(j) >= s(j + 1));
        }
        Tensor3 hat(5, 4, 3);
        for (Index i = 0; i < 3; ++i) {
            const auto u = (size_t)i;
            Matrix US = F.Uhat[u];
            for (Index j = 0; j < 3; ++j)
                for (Index r = 0; r < 5; ++r) US(r, j) *= F.shat[u](j);
            hat.set_slice(i, US * F.Vhat[u].transpose());
        }
        Tensor3 recon = tsvdq_reconstruct(F);
        CHECK(frobenius_norm(mode3_product(hat, T.Q) - recon) <= 1e-12 * frobenius_norm(recon));
        check_throws<argument_error>([&] { tsvdq(A, T, 0); }, "k=0");
        check_throws<argument_error>([&] { tsvdq(A, T, 5); }, "k=5");
    }
    // test_decompositions.cpp:80-103 — limits
    {
        Tensor3 A = seeded(4, 3, 5, 42);
        Transform full = random_orthogonal_transform(5, 5, 9);
        TsvdqFactors Ff = tsvdq(A, full, 3);
        CHECK(frobenius_norm(A - tsvdq_reconstruct(Ff)) <= 1e-10 * frobenius_norm(A));
        Transform part = random_orthogonal_transform(5, 3, 9);
        Tensor3 proj = mode3_product(A, part.Q * part.Q.transpose());
        CHECK(frobenius_norm(proj - tsvdq_reconstruct(tsvdq(A, part, 3))) <= 1e-10 * frobenius_norm(A));
    }
    // test_star_products.cpp:90-102 — scale law
    {
        Tensor3 A = seeded(2, 2, 4, 8), B = seeded(2, 3, 4, 9);
        Transform unit = dct_transform(4, 2);
        Tensor3 base = star_q_product(A, B, StarContext(unit));
        for (double c : {-2.0, 0.5, 3.0}) {
            Tensor3 got = star_q_product(A, B, StarContext(custom_transform(unit.Q, c)));
            CHECK(frobenius_norm(got - c * base) <= 1e-12 * std::fabs(c) * frobenius_norm(base));
        }
    }
    // test_star_products.cpp:185-206 — transpose rule
    {
        Tensor3 A = seeded(3, 2, 5, 10), B = seeded(2, 4, 5, 11);
        StarContext ctx(random_orthogonal_transform(5, 3, 13));
        Tensor3 lhs = star_q_transpose(star_q_product(A, B, ctx), ctx);
        Tensor3 rhs = star_q_product(star_q_transpose(B, ctx), star_q_transpose(A, ctx), ctx);
        CHECK(lhs.n1() == 4 && lhs.n2() == 3);
        CHECK(frobenius_norm(lhs - rhs) <= 1e-12 * frobenius_norm(lhs));
    }
    // test_decompositions.cpp:118-124 — star_q_rank
    CHECK(star_q_rank(counterexample(), identity_transform(2, 2)) == 2);
    CHECK(star_q_rank(counterexample(), haar_transform(2, 1)) == 1);
    CHECK(star_q_rank(Tensor3(3, 3, 4), dct_transform(4, 2)) == 0);
    // test_matrix_kernels.cpp:11-35 — SVD contract and pins
    {
        Matrix A(2, 2);
        A(0, 0) = s2;
        SvdResult d = svd(A);
        CHECK(std::fabs(d.s(0) - s2) <= 1e-14 * s2 && std::fabs(d.s(1)) <= 1e-14);
        SvdResult di = svd(Matrix::Identity(3, 3));
        for (Index j = 0; j < 3; ++j) CHECK(std::fabs(di.s(j) - 1.0) <= 1e-14);
        check_throws<argument_error>([&] { truncated_svd(A, 3); }, "truncated k");
        Matrix Q = orthonormalize(Matrix::Identity(4, 2) + 0.1 * Matrix::Identity(4, 2));
        CHECK((Q.transpose() * Q - Matrix::Identity(2, 2)).norm() <= 1e-12);
    }
    // test_decompositions.cpp:126-146 — tsvdq2 keeps everything at gamma = 1
    {
        Tensor3 A = seeded(4, 5, 6, 44);
        Transform T = dct_transform(6, 4);
        TsvdqIIFactors F = tsvdq2(A, T, 1.0);
        Tensor3 Ahat = mode3_product(A, T.Q.transpose());
        for (Index i = 0; i < 4; ++i)
            CHECK(F.multirank[(size_t)i] == numerical_rank(svd(Ahat.slice(i)).s, kDefaultRankTol));
        ApproxError e = tsvdq2_error(A, F);
        CHECK(std::fabs(e.total - projection_error(A, T)) <= 1e-10 * frobenius_norm(A));
        CHECK(e.eckart_young <= 1e-10 * frobenius_norm(A));
        check_throws<argument_error>([&] { tsvdq2(A, T, 0.0); }, "gamma 0");
        check_throws<argument_error>([&] { tsvdq2(A, T, 1.5); }, "gamma 1.5");
    }
    // test_decompositions.cpp:148-160 — tie-break on the 2x2x2 fixture
    {
        TsvdqIIFactors F = tsvdq2(counterexample(), identity_transform(2, 2), 0.5);
        CHECK(F.implicit_rank() == 2 && F.multirank[0] == 2 && F.multirank[1] == 0);
        ApproxError e = tsvdq2_error(counterexample(), F);
        CHECK(std::fabs(e.total * e.total - 2.0) <= 1e-12);
    }
    // test_decompositions.cpp:162-177 — exact-rank slices reproduce tsvdq
    {
        Transform T = dct_transform(5, 3);
        Tensor3 Ahat(4, 4, 3);  // rank-2 transform-domain slices, lifted by Q
        for (Index i = 0; i < 3; ++i) {
            Tensor3 u = seeded(4, 2, 1, 60 + (unsigned)i), v = seeded(4, 2, 1, 70 + (unsigned)i);
            Matrix m(4, 4);
            for (Index a = 0; a < 4; ++a)
                for (Index b = 0; b < 4; ++b)
                    m(a, b) = u(a, 0, 0) * v(b, 0, 0) + u(a, 1, 0) * v(b, 1, 0);
            Ahat.set_slice(i, m);
        }
        Tensor3 A = mode3_product(Ahat, T.Q);
        TsvdqIIFactors F2 = tsvdq2(A, T, 1.0);
        for (Index r : F2.multirank) CHECK(r == 2);
        TsvdqFactors F1 = tsvdq(A, T, 2);
        CHECK(frobenius_norm(tsvdq2_reconstruct(F2) - tsvdq_reconstruct(F1)) <= 1e-12 * frobenius_norm(A));
        CHECK(std::fabs(tsvdq2_error(A, F2).total - tsvdq_error(A, F1).total) <= 1e-12 * frobenius_norm(A));
    }
    // test_decompositions.cpp:179-188 — full transform, gamma = 1: lossless
    {
        Tensor3 A = seeded(3, 4, 4, 46);
        ApproxError e = tsvdq2_error(A, tsvdq2(A, dct_transform(4, 4), 1.0));
        const double sc = frobenius_norm(A);
        CHECK(e.total <= 1e-10 * sc && e.eckart_young <= 1e-10 * sc && e.projection <= 1e-10 * sc);
    }
    // test_decompositions.cpp:190-205 — error decomposition on random instances
    for (int i = 0; i < 10; ++i) {
        Tensor3 A = seeded(4, 3, 5, 470 + (unsigned)i);
        Transform T = random_orthogonal_transform(5, 3, 100 + (uint64_t)i);
        TsvdqIIFactors F = tsvdq2(A, T, 0.8);
        ApproxError e = tsvdq2_error(A, F);
        const double lhs = e.total * e.total,
                     rhs = e.eckart_young * e.eckart_young + e.projection * e.projection;
        CHECK(std::fabs(lhs - rhs) <= 1e-10 * lhs);
        CHECK(std::fabs(e.total - frobenius_norm(A - tsvdq2_reconstruct(F))) <= 1e-10 * frobenius_norm(A));
    }
    // test_io.cpp:50-112 — PT3 round trip, matrix container, malformed files
    {
        namespace fs = std::filesystem;
        const fs::path f = fs::temp_directory_path() / ("ppc_io_" + std::to_string(::getpid()) + ".pt3");
        Tensor3 A = seeded(4, 3, 5, 71);
        write_pt3(f, A);
        Tensor3 B = read_pt3(f);
        CHECK(B.n1() == 4 && B.n2() == 3 && B.n3() == 5);
        CHECK(std::memcmp(A.data(), B.data(), sizeof(double) * (size_t)A.size()) == 0);
        Matrix M = seeded(3, 7, 1, 5).slice(0);
        write_pt3_matrix(f, M);
        Matrix R = read_pt3_matrix(f);
        CHECK(R.rows() == 3 && R.cols() == 7 && (M - R).norm() == 0.0);
        write_pt3(f, seeded(2, 2, 2, 72));
        std::vector<char> good;
        {
            std::ifstream in(f, std::ios::binary);
            good.assign(std::istreambuf_iterator<char>(in), {});
        }
        auto spew = [&](const std::vector<char>& b) {
            std::ofstream out(f, std::ios::binary | std::ios::trunc);
            out.write(b.data(), (std::streamsize)b.size());
        };
        for (auto [off, val] : std::vector<std::pair<size_t, char>>{{0, 'X'}, {4, 9}, {8, 7}}) {
            std::vector<char> b = good;
            b[off] = val;
            spew(b);
            check_throws<format_error>([&] { read_pt3(f); }, "tampered header");
        }
        {
            std::vector<char> b = good;
            b.pop_back();
            spew(b);
            check_throws<format_error>([&] { read_pt3(f); }, "truncated");
            b = good;
            b.push_back(0);
            spew(b);
            check_throws<format_error>([&] { read_pt3(f); }, "trailing");
            b = good;
            for (size_t i = 12; i < 20; ++i) b[i] = '\xff';
            spew(b);
            check_throws<format_error>([&] { read_pt3(f); }, "overflow");
            b = good;
            for (size_t i = 12; i < 20; ++i) b[i] = 0;
            spew(b);
            check_throws<format_error>([&] { read_pt3(f); }, "zero extent");
        }
        check_throws<format_error>([&] { read_pt3(f.string() + ".does-not-exist"); }, "missing");
        fs::remove(f);
    }
    // test_star_products.cpp:34-68 — star_m
    {
        Tensor3 a = make_tube({2, 4, 6, 8}), b = make_tube({1, -1, 1, 0});
        Tensor3 ab = star_m_product(a, b, haar_transform(4, 4).Q.transpose());
        const double want[4] = {2, 4, 3, 8};
        for (Index k = 0; k < 4; ++k) CHECK(std::fabs(ab(0, 0, k) - want[k]) <= 1e-12);
        Tensor3 e = star_m_product(make_tube({1, 2, 3}), make_tube({4, -5, 0.5}), Matrix::Identity(3, 3));
        CHECK(std::fabs(e(0, 0, 0) - 4) <= 1e-14 && std::fabs(e(0, 0, 1) + 10) <= 1e-14 &&
              std::fabs(e(0, 0, 2) - 1.5) <= 1e-14);
        Matrix singular(2, 2);
        singular(0, 0) = 1.0;
        check_throws<degenerate_input_error>([&] { star_m_product(make_tube({1, 2}), make_tube({1, 2}), singular); },
                                             "singular M");
        check_throws<shape_error>([&] { star_m_product(make_tube({1, 2}), make_tube({1, 2, 3}), Matrix::Identity(2, 2)); },
                                  "star_m shapes");
    }
    // test_decompositions.cpp:203-255 — hosvd and the matrix SVD baseline
    {
        Tensor3 A = seeded(4, 3, 5, 48);
        HosvdFactors F = hosvd(A, 4, 3, 5);
        CHECK(frobenius_norm(A - hosvd_reconstruct(F)) <= 1e-10 * frobenius_norm(A));
        CHECK((F.U1.transpose() * F.U1 - Matrix::Identity(4, 4)).norm() <= 1e-10 * 4);
        HosvdFactors Fc = hosvd(counterexample(), 2, 2, 1);
        const double err = frobenius_norm(counterexample() - hosvd_reconstruct(Fc));
        CHECK(std::fabs(err * err - 2.0) <= 1e-12);
        check_throws<argument_error>([&] { hosvd(A, 0, 1, 1); }, "hosvd k1");
        check_throws<argument_error>([&] { hosvd(A, 1, 4, 1); }, "hosvd k2");
        Tensor3 B = seeded(3, 4, 5, 49);
        CHECK(matrix_svd_baseline(B, 4).error <= 1e-10 * frobenius_norm(B));
        MatrixSvdBaseline mb = matrix_svd_baseline(counterexample(), 1);
        CHECK(mb.factors.s.size() == 1 && std::fabs(mb.factors.s(0) - s2) <= 1e-12);
        CHECK(std::fabs(mb.error * mb.error - 2.0) <= 1e-12);
        CHECK(matrix_svd_baseline(Tensor3(2, 3, 2), 2).error == 0.0);
        check_throws<argument_error>([&] { matrix_svd_baseline(B, 0); }, "msvd k0");
        check_throws<argument_error>([&] { matrix_svd_baseline(B, 5); }, "msvd k5");
    }
    // errors: argument / shape / degenerate
    check_throws<argument_error>([&] { identity_transform(4, 9); }, "p > n3");
    check_throws<argument_error>([&] { haar_transform(3, 2); }, "haar n3");
    check_throws<shape_error>([&] { Tensor3(0, 3, 5); }, "extent");
    check_throws<degenerate_input_error>([&] { custom_transform(Matrix(4, 2)); }, "stiefel");
    std::printf("%d/%d checks passed\n", g_checks - g_fail, g_checks);
    return g_fail ? 1 : 0;
}
