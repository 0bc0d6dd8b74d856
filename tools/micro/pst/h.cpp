#include <dlfcn.h>
#include <chrono>
#include <cstdio>
#include <cstdarg>
int ctk_fail(int code, const char* fmt, ...) { return code; }
#include "../../../paper_2602_17892_b200/csrc/ctk_host.cpp"
#include <random>
int main() {
    void* h = dlopen("/opt/prime-rl/.venv/lib/python3.12/site-packages/scipy.libs/libscipy_openblas-5f890258.so", RTLD_NOW);
    void* f = dlsym(h, "scipy_dbdsqr_"); if (!f) f = dlsym(h, "dbdsqr_");
    printf("dbdsqr %p\n", f);
    ctk_set_lapack_extra(f);
    std::mt19937_64 rng(0); std::normal_distribution<double> nd;
    for (int k : {40, 80, 40, 80}) {
        int m = k + 1, n = k;
        std::vector<double> H((size_t)m * n, 0.0);
        for (int i = 0; i < m; ++i) for (int j = 0; j < n; ++j) if (i <= j + 1) H[(size_t)i * n + j] = nd(rng);
        Bidiag bd;
        auto t0 = std::chrono::steady_clock::now();
        for (int it = 0; it < 200; ++it) bidiagonalize(H.data(), m, n, 2.0, bd);
        auto t1 = std::chrono::steady_clock::now();
        std::vector<double> sv, ee, c, work(4 * n + 4);
        for (int it = 0; it < 200; ++it) {
            sv = bd.d; ee = bd.e; c.assign(bd.g.begin(), bd.g.begin() + n);
            char uplo = 'U'; int nn = n, ncvt = 0, nru = 0, ncc = 1, ldvt = 1, ldu = 1, ldc = n, info = 0; double dummy = 0;
            g_dbdsqr(&uplo, &nn, &ncvt, &nru, &ncc, sv.data(), ee.data(), &dummy, &ldvt, &dummy, &ldu, c.data(), &ldc, work.data(), &info);
        }
        auto t2 = std::chrono::steady_clock::now();
        double lam = 0; 
        for (int it = 0; it < 200; ++it) select_sc(sv.data(), c, k, m, 2.0, S_GCV, 200, &lam);
        auto t3 = std::chrono::steady_clock::now();
        std::vector<double> z(n), y(n);
        for (int it = 0; it < 200; ++it) {
            std::vector<double> gn(bd.g.begin(), bd.g.begin() + n);
            damped_bidiag_solve(bd.d, std::vector<double>(bd.e.begin(), bd.e.begin() + n - 1), gn, 0.1, sv[0], m, z.data());
            apply_p(bd, z.data(), y.data());
        }
        auto t4 = std::chrono::steady_clock::now();
        auto us = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count() / 200 * 1e6; };
        printf("k=%d bidiag %.1f us, dbdsqr %.1f us, select %.1f us, solve %.1f us\n", k, us(t0, t1), us(t1, t2), us(t2, t3), us(t3, t4));
    }
}
