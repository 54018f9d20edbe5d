// CUDA-free host copy helpers shared by the C ABI (shtc.cu, group.cu, through hostutil.h) and
// the C++ drop-in (sht_dropin.cpp): a persistent host worker pool, streaming-store copies, and
// fast value-initialised result containers.
#pragma once

#include <immintrin.h>
#include <sys/mman.h>

#include <algorithm>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace shtc_host {

// Persistent host worker pool for the staging copies (process-wide; threads start on first use
// and park on a condition variable between jobs).
class CopyPool {
public:
    static CopyPool& get() {
        static CopyPool pool;
        return pool;
    }
    unsigned size() const { return (unsigned)workers_.size() + 1; }
    // run fn(i) for i in [0, n) on the workers and the calling thread; returns when all are done
    void run(unsigned n, const std::function<void(unsigned)>& fn) {
        std::unique_lock<std::mutex> job_lock(job_mu_);  // one job at a time
        {
            std::lock_guard<std::mutex> lk(mu_);
            fn_ = &fn;
            n_ = n;
            next_ = 1;  // index 0 runs on the caller
            pending_ = n - 1;
            ++gen_;
        }
        cv_.notify_all();
        fn(0);
        for (;;) {  // the caller takes pieces too
            unsigned i;
            {
                std::lock_guard<std::mutex> lk(mu_);
                if (next_ >= n_) break;
                i = next_++;
            }
            fn(i);
            std::lock_guard<std::mutex> lk(mu_);
            if (--pending_ == 0) done_.notify_all();
        }
        std::unique_lock<std::mutex> lk(mu_);
        done_.wait(lk, [&] { return pending_ == 0; });
        fn_ = nullptr;
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
            ++gen_;
        }
        cv_.notify_all();
        for (auto& t : workers_) t.join();
    }

private:
    CopyPool() {
        unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
        if (const char* e = std::getenv("SHTC_COPY_THREADS")) hw = std::max(1, std::atoi(e));
        for (unsigned i = 1; i < hw; ++i) workers_.emplace_back([this] { loop(); });
    }
    void loop() {
        unsigned seen = 0;
        for (;;) {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] { return stop_ || (gen_ != seen && fn_ && next_ < n_); });
            if (stop_) return;
            seen = gen_;
            while (fn_ && next_ < n_) {
                const unsigned i = next_++;
                const std::function<void(unsigned)>* fn = fn_;
                lk.unlock();
                (*fn)(i);
                lk.lock();
                if (--pending_ == 0) done_.notify_all();
            }
        }
    }
    std::vector<std::thread> workers_;
    std::mutex mu_, job_mu_;
    std::condition_variable cv_, done_;
    const std::function<void(unsigned)>* fn_ = nullptr;
    unsigned n_ = 0, next_ = 0, pending_ = 0, gen_ = 0;
    bool stop_ = false;
};

// memcpy on all host cores (pageable <-> staging copies are bound by host memory bandwidth)
// Large copies with non-temporal (streaming) AVX2 stores: the destination lines are not read
// for ownership first, which cuts the host memory traffic of a staging copy by a third.
__attribute__((target("avx2"))) inline void nt_memcpy(void* dst, const void* src, size_t n) {
    char* d = static_cast<char*>(dst);
    const char* s = static_cast<const char*>(src);
    size_t i = 0;
    while (i < n && (reinterpret_cast<uintptr_t>(d + i) & 31)) {
        d[i] = s[i];
        ++i;
    }
    for (; i + 128 <= n; i += 128) {
        const __m256d a = _mm256_loadu_pd(reinterpret_cast<const double*>(s + i));
        const __m256d b = _mm256_loadu_pd(reinterpret_cast<const double*>(s + i + 32));
        const __m256d c = _mm256_loadu_pd(reinterpret_cast<const double*>(s + i + 64));
        const __m256d e = _mm256_loadu_pd(reinterpret_cast<const double*>(s + i + 96));
        _mm256_stream_pd(reinterpret_cast<double*>(d + i), a);
        _mm256_stream_pd(reinterpret_cast<double*>(d + i + 32), b);
        _mm256_stream_pd(reinterpret_cast<double*>(d + i + 64), c);
        _mm256_stream_pd(reinterpret_cast<double*>(d + i + 96), e);
    }
    _mm_sfence();
    if (i < n) std::memcpy(d + i, s + i, n - i);
}

inline void piece_copy(void* dst, const void* src, size_t bytes) {
    static const bool nt = [] {
        const char* e = std::getenv("SHTC_COPY_NT");
        return (e ? std::atoi(e) != 0 : true) && __builtin_cpu_supports("avx2");
    }();
    if (nt && bytes >= (size_t(1) << 16)) nt_memcpy(dst, src, bytes);
    else std::memcpy(dst, src, bytes);
}

inline void par_memcpy(void* dst, const void* src, size_t bytes) {
    CopyPool& pool = CopyPool::get();
    const size_t min_piece = size_t(2) << 20;
    const unsigned nt = (unsigned)std::max<size_t>(1, std::min<size_t>(pool.size(), bytes / min_piece));
    if (nt <= 1) {
        piece_copy(dst, src, bytes);
        return;
    }
    const size_t piece = (bytes / nt + 63) & ~size_t(63);
    pool.run(nt, [&](unsigned i) {
        const size_t b = std::min(bytes, piece * i), e = i + 1 == nt ? bytes : std::min(bytes, piece * (i + 1));
        if (e > b) piece_copy(static_cast<char*>(dst) + b, static_cast<const char*>(src) + b, e - b);
    });
}


// A std::vector<T> of n value-initialised elements (the containers the reference API returns by
// value) without the page-fault-bound single-thread first touch: the storage is reserved,
// advised for transparent huge pages, touched on all host cores, and only then value-
// initialised (now a memory-bound memset).  C4 map (403 MB) on the GPU box: 147-160 ms for
// std::vector<double>(n, 0.0), 36-41 ms this way (tools/alloc_probe.cpp).
template <class T>
void value_init(std::vector<T>& v, size_t n) {
    v.clear();
    v.reserve(n);
    const size_t bytes = n * sizeof(T);
    if (bytes >= (size_t(8) << 20)) {
        const uintptr_t b = (reinterpret_cast<uintptr_t>(v.data()) + 4095) & ~uintptr_t(4095);
        const uintptr_t e = (reinterpret_cast<uintptr_t>(v.data()) + bytes) & ~uintptr_t(4095);
        if (e > b) madvise(reinterpret_cast<void*>(b), e - b, MADV_HUGEPAGE);
        // own threads, not the copy pool: this runs beside a transform whose staging copies use it
        char* p = reinterpret_cast<char*>(v.data());  // raw storage, no element constructed yet
        const unsigned nt = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
        const size_t piece = (bytes / nt + 4095) & ~size_t(4095);
        std::vector<std::thread> th;
        for (unsigned i = 0; i < nt; ++i)
            th.emplace_back([=] {
                const size_t lo = std::min(bytes, piece * i), hi = std::min(bytes, piece * (i + 1));
                for (size_t o = lo; o < hi; o += 4096) p[o] = 0;  // first touch of each page
            });
        for (auto& t : th) t.join();
    }
    v.resize(n);
}

}  // namespace shtc_host
