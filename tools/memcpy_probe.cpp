// Host copy rate on the GPU box: 403 MB pageable -> page-locked-like buffer on T threads with
// std::memcpy against non-temporal (streaming) AVX2 stores -- the staging copies of the
// pageable-buffer entry points are host-memory bound.
//
//   g++ -O2 -pthread tools/memcpy_probe.cpp -o tools/memcpy_probe.bin
#include <immintrin.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

__attribute__((target("avx2"))) static void nt_copy(char* d, const char* s, size_t n) {
    size_t i = 0;
    while (i < n && (reinterpret_cast<uintptr_t>(d + i) & 31)) { d[i] = s[i]; ++i; }
    for (; i + 128 <= n; i += 128) {
        __m256d a = _mm256_loadu_pd(reinterpret_cast<const double*>(s + i));
        __m256d b = _mm256_loadu_pd(reinterpret_cast<const double*>(s + i + 32));
        __m256d c = _mm256_loadu_pd(reinterpret_cast<const double*>(s + i + 64));
        __m256d e = _mm256_loadu_pd(reinterpret_cast<const double*>(s + i + 96));
        _mm256_stream_pd(reinterpret_cast<double*>(d + i), a);
        _mm256_stream_pd(reinterpret_cast<double*>(d + i + 32), b);
        _mm256_stream_pd(reinterpret_cast<double*>(d + i + 64), c);
        _mm256_stream_pd(reinterpret_cast<double*>(d + i + 96), e);
    }
    _mm_sfence();
    for (; i < n; ++i) d[i] = s[i];
}

template <class F>
static double run(int nt, size_t bytes, F f) {
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    const size_t piece = (bytes / nt + 63) & ~size_t(63);
    for (int i = 0; i < nt; ++i)
        th.emplace_back([&, i] {
            const size_t b = std::min(bytes, piece * i), e = i + 1 == nt ? bytes : std::min(bytes, piece * (i + 1));
            if (e > b) f(b, e - b);
        });
    for (auto& t : th) t.join();
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

int main() {
    const size_t bytes = 403ull << 20;
    char* s = (char*)aligned_alloc(64, bytes);
    char* d = (char*)aligned_alloc(64, bytes);
    memset(s, 1, bytes);
    memset(d, 2, bytes);
    printf("avx2 %d avx512f %d\n", __builtin_cpu_supports("avx2"), __builtin_cpu_supports("avx512f"));
    for (int nt : {4, 8, 16}) {
        double best_m = 1e9, best_n = 1e9;
        for (int r = 0; r < 4; ++r) {
            best_m = std::min(best_m, run(nt, bytes, [&](size_t b, size_t n) { memcpy(d + b, s + b, n); }));
            best_n = std::min(best_n, run(nt, bytes, [&](size_t b, size_t n) { nt_copy(d + b, s + b, n); }));
        }
        printf("threads %2d: memcpy %.2f ms (%.1f GB/s)  nt-store %.2f ms (%.1f GB/s)\n", nt, best_m, bytes / best_m / 1e6,
               best_n, bytes / best_n / 1e6);
    }
    return 0;
}
