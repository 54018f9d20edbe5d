// Cost of the containers the reference API returns by value (std::vector<double> of 403 MB, the
// C4 SkyMap) on the GPU box: plain value-initialisation against a parallel first touch of the
// reserved storage (with and without MADV_HUGEPAGE) before the resize.
//
//   g++ -O2 -pthread tools/alloc_probe.cpp -o tools/alloc_probe.bin
#include <sys/mman.h>
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

static double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static void par_touch(char* p, size_t bytes, int nt) {
    std::vector<std::thread> th;
    const size_t piece = (bytes / nt + 4095) & ~size_t(4095);
    for (int i = 0; i < nt; ++i)
        th.emplace_back([=] {
            const size_t b = std::min(bytes, piece * i), e = std::min(bytes, piece * (i + 1));
            if (e > b) std::memset(p + b, 0, e - b);
        });
    for (auto& t : th) t.join();
}

int main() {
    std::FILE* f = std::fopen("/sys/kernel/mm/transparent_hugepage/enabled", "r");
    char buf[256] = {0};
    if (f) {
        if (!std::fgets(buf, sizeof buf, f)) buf[0] = 0;
        std::fclose(f);
    }
    std::printf("THP: %s", buf);
    const size_t n = 50331648;  // C4 pixels
    for (int rep = 0; rep < 3; ++rep) {
        double t0 = now_ms();
        { std::vector<double> v(n, 0.0); v[n / 2] = 1; }
        double t1 = now_ms();
        double tp = 0, tr = 0;
        {
            std::vector<double> v;
            v.reserve(n);
            const double a = now_ms();
            par_touch(reinterpret_cast<char*>(v.data()), n * 8, 16);
            const double b = now_ms();
            v.resize(n);
            tr = now_ms() - b;
            tp = b - a;
        }
        double t2 = now_ms();
        double hp = 0, hr = 0;
        {
            std::vector<double> v;
            v.reserve(n);
            const double a = now_ms();
            madvise(reinterpret_cast<void*>(reinterpret_cast<uintptr_t>(v.data()) & ~uintptr_t(4095)), n * 8, MADV_HUGEPAGE);
            par_touch(reinterpret_cast<char*>(v.data()), n * 8, 16);
            const double b = now_ms();
            v.resize(n);
            hr = now_ms() - b;
            hp = b - a;
        }
        double t3 = now_ms();
        std::printf("vector(n, 0): %.1f ms | reserve + parallel touch %.1f + resize %.1f = %.1f ms | + MADV_HUGEPAGE: %.1f + %.1f = %.1f ms\n",
                    t1 - t0, tp, tr, t2 - t1, hp, hr, t3 - t2);
    }
    return 0;
}
