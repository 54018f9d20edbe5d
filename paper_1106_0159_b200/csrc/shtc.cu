// libshtc: C ABI (include/shtc.h) over the sm_100a SHT kernels.
//
// Host-side responsibilities (all C++, no Python on the path):
//   * geometry / band state, stream (ring-pair) construction   grid.cpp:133-151 semantics
//   * log(mu_m) with glibc lgamma and per-stream log2(1-x^2)     legendre.cpp:16-20, 62-76
//     (kept on the host so the seeds match the reference bit for bit)
//   * Legendre plan: recurrence tables + activation scan + alive-tile lists ordered by cost
//   * ring-FFT plan: per-ring descriptors, twiddle/chirp tables, size classes
//   * validation with the reference's error classes (transforms.cpp:222-242, 338-345, 403-455)
// There is no CPU fallback: every compute entry point needs the CUDA device.

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <numeric>
#include <string>
#include <tuple>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <functional>
#include <vector>

#include "../../include/shtc.h"
#include "common.cuh"
#include "kernels.h"
#include "hostutil.h"

using namespace shtk;
using shtc_host::host_pinned;
using shtc_host::par_memcpy;
using shtc_host::CopyPool;

namespace {

thread_local std::string g_last_error;

struct ShtcError {
    shtc_status code;
    std::string msg;
};

[[noreturn]] void fail(shtc_status c, const std::string& m) { throw ShtcError{c, m}; }

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        fail(e == cudaErrorMemoryAllocation ? SHTC_ENOMEM : SHTC_ECUDA,
             std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(x) cuda_check((x), #x)

// Page-locked host staging buffer (cudaHostAlloc), grown on demand and kept by the context.
struct PinnedBuf {
    void* p = nullptr;
    size_t bytes = 0;
    PinnedBuf() = default;
    PinnedBuf(const PinnedBuf&) = delete;
    PinnedBuf& operator=(const PinnedBuf&) = delete;
    ~PinnedBuf() { release(); }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        bytes = 0;
    }
    void ensure(size_t b) {
        if (b <= bytes && p) return;
        release();
        CK(cudaHostAlloc(&p, b ? b : 16, cudaHostAllocDefault));
        bytes = b;
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; o.bytes = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p;
            bytes = o.bytes;
            o.p = nullptr;
            o.bytes = 0;
        }
        return *this;
    }
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    void ensure(size_t b) {
        if (b <= bytes && p) return;
        release();
        if (b == 0) b = 16;
        CK(cudaMalloc(&p, b));
        bytes = b;
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
    template <class T>
    void upload(const std::vector<T>& v, cudaStream_t s) {
        ensure(v.size() * sizeof(T));
        if (!v.empty()) CK(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
    }
};

constexpr double kLn2 = 0.69314718055994530942;
constexpr double kLn4Pi = 2.5310242469692907930;  // legendre.cpp:9

// log(mu_m), the reference expression verbatim (legendre.cpp:16-20).
double host_log_mu(int m) {
    return -m * kLn2 - std::lgamma(m + 1.0) + 0.5 * (std::lgamma(2.0 * m + 2.0) - kLn4Pi);
}

struct Stream {
    double x;
    int north, south;
};

struct LegPlan {
    bool built = false;
    int lmax = -1;
    std::vector<int> ms;
    std::vector<Stream> streams;
    DevBuf ms_d, logmu_d, sx, sl2, spos, sn, ss, tab_off, A, C, T, tile_info, tile_list, tile_off,
        tile_cnt, a2m_items, m2a_items, m2a_per_m, m2a_slot, m2a_scratch, counters, ck_q, ck_act,
        a2m_items_band, m2a_items_band, m2a_per_m_band, m2a_slot_band;
    uint64_t prefix_steps = 0, checked_steps = 0, fast_steps = 0;
    // Pipelined host-buffer paths (see shtc_alm2map): latitude bands of tiles, numbered from
    // the equator.  alm2map launches: band tc's items (band 0 also split by order chunk mc so
    // it can start while a_lm is still arriving); map2alm launches: band tc's items (the last
    // band also split by order chunk so the a_lm copies start before it ends); after map2alm
    // launch j the orders whose last item was in launch j are final (runs of order indices).
    struct PipeLaunch {
        int tc, mc, begin, end;
    };
    std::vector<int> chunk_mi;  // order chunk k = order indices [chunk_mi[k], chunk_mi[k+1])
    std::vector<PipeLaunch> a2m_launch;  // ranges of the band-ordered item lists
    std::vector<PipeLaunch> m2a_launch;
    LegPlanView band_view{};             // view with the band-ordered item lists
    std::vector<std::vector<std::pair<int, int>>> m2a_done;  // per m2a launch: final order runs
    DevBuf m2a_final_list;           // order indices final after each m2a launch, concatenated
    std::vector<int> m2a_final_off;  // launch j: [m2a_final_off[j], m2a_final_off[j+1])
    LegPlanView view{};
    // executed: map2alm passes (tile pairs); executed_a2m: alm2map (single tiles)
    uint64_t nominal = 0, executed = 0, executed_a2m = 0, useful = 0;
    int m2a_group = LEG_M2A_GROUP;  // tiles per map2alm item of the device-resident set
    double build_ms = 0.0;
};

// pipelined host-buffer entry points: latitude bands (ring stage + Legendre units, pixel
// copies) and order chunks (a_lm copies)
constexpr int kMaxPipeBands = 16;
// SHTC_PIPE_BANDS overrides the band count (experiments)
// 6 bands: with the round-2 kernels the C4 pair from pinned memory measured 22.59 ms against
// 22.80 ms for 8 (map2alm 11.88 vs 12.20; alm2map 10.71 vs 10.60), 10 and 12 slower
// (tools/pipe_bands.sh, tools/pipe_bands_w.sh)
int pipe_bands() {
    static const int b = std::getenv("SHTC_PIPE_BANDS")
                             ? std::min(kMaxPipeBands, std::max(1, std::atoi(std::getenv("SHTC_PIPE_BANDS"))))
                             : 6;
    return b;
}
#define kPipeBands pipe_bands()
// a_lm order chunks of the alm2map head (SHTC_A2M_CHUNKS overrides)
int order_chunks() {
    static const int c = std::getenv("SHTC_A2M_CHUNKS") ? std::min(16, std::max(1, std::atoi(std::getenv("SHTC_A2M_CHUNKS")))) : 4;
    return c;
}
#define kOrderChunks order_chunks()
constexpr int kPipeEvents = 128;
// side streams of the ring stage: each small-ring class launch (latency bound, few CTAs busy)
// gets its own, so their latencies overlap (a worker's share of polar rings is all small
// classes)
constexpr int kFftAux = 6;
// SHTC_FFT_AUX overrides the count (1..kFftAux).  Tests that run several workers' contexts in
// one process with device-side barriers use fewer, so that every context's streams keep their
// own hardware queue (CUDA_DEVICE_MAX_CONNECTIONS <= 32): a spinning barrier kernel must never
// share a queue with another worker's pending kernel
int fft_aux_count() {
    static const int n = std::getenv("SHTC_FFT_AUX") ? std::min(kFftAux, std::max(1, std::atoi(std::getenv("SHTC_FFT_AUX"))))
                                                      : kFftAux;
    return n;
}

struct FftPlan {
    bool built = false;
    int mmax = -1;  // the phase-factor tables cover orders 0..mmax
    DevBuf descs[FFT_N_CLASSES];
    int count[FFT_N_CLASSES] = {};
    // latitude bands of the pipelined paths: class c's descriptors of band k are
    // [range_start[c][k], range_start[c][k+1]); band k covers the pixel intervals band_pix[k]
    std::vector<int> range_start[FFT_N_CLASSES];
    std::vector<std::vector<std::pair<int64_t, int64_t>>> band_pix;
    DevBuf tabs;
    DevBuf counters;  // ring queues of the power-of-two engine's launches (one per class)
    int64_t tw_off[FFT_N_CLASSES] = {};  // twiddle table of each power-of-two class
    int alt[FFT_N_CLASSES] = {};         // class runs its alternative kernel (RingStageArgs::alt)
    double build_ms = 0.0;
};

}  // namespace

struct shtc_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t own_stream = nullptr;
    std::string err;
    // grid
    int n_rings = 0;
    std::vector<double> cos_theta, phi0, weight;
    std::vector<int> nphi;
    std::vector<int64_t> pixoff;
    int64_t npix = 0;
    bool symmetric = false, mirror = true, grid_set = false;
    // band
    int lmax = -1, mmax = -1;
    std::vector<int> ms;
    bool band_set = false;
    std::vector<double> log_mu;
    bool ladder = true;  // ScaleLadder::standard (false: ScaleLadder::unscaled)
    // exchange layout (stage API)
    bool custom_layout = false;
    std::vector<int64_t> row_off;
    std::vector<int> ring_list;
    std::vector<int64_t> m_base, m_stride;
    DevBuf row_off_d, m_base_d, m_stride_d;
    DevBuf m_order_d;  // the orders by m_base: each owner's block contiguous (analysis unfold)
    // synthesis-direction override (shtc_set_exchange_layout_synthesis): order-major blocks
    bool syn_layout = false;
    DevBuf syn_row_off_d, syn_row_stride_d, syn_m_base_d, syn_m_stride_d;
    // fused exchange over peer memory: per-ring row / per-order column addresses in the
    // owners' buffers (valid on this device: NVLink peer mappings or CUDA IPC)
    DevBuf peer_row_ptr, peer_col_ptr;
    bool peers_set = false;
    // identity layout for whole transforms
    DevBuf id_row_off, id_m_base, id_m_stride;
    // plans
    LegPlan leg;
    FftPlan fft_id;      // identity ring list
    FftPlan fft_custom;  // custom ring list
    // operator-API plan cache
    LegPlan op_leg;
    std::vector<double> op_x;
    // scratch
    DevBuf delta, alm_buf, map_buf, stats;
    PinnedBuf stage_alm, stage_map;  // staging of pageable host buffers (host-buffer entry points)
    cudaEvent_t ev[8] = {};
    // pipelined host-buffer paths: copy streams, two Legendre streams (consecutive launches
    // alternate so one launch's tail overlaps the next) and a high-priority ring-stage stream
    cudaStream_t h2d = nullptr, d2h = nullptr, lst[2] = {}, fst = nullptr;
    cudaEvent_t pev[kPipeEvents] = {};  // ordering events
    cudaEvent_t tev[kPipeEvents] = {};  // timing events
    // ring stage: the small-ring classes run on side streams beside the large ones
    cudaStream_t fft_aux[kFftAux] = {};
    cudaEvent_t fft_fork = nullptr, fft_join[kFftAux] = {};
};

namespace {

bool is_smooth7(int n) {
    for (int p : {2, 3, 5, 7})
        while (n % p == 0) n /= p;
    return n == 1;
}

std::vector<int> radix_plan(int B) {
    std::vector<int> r;
    int n = B;
    while (n % 8 == 0) { r.push_back(8); n /= 8; }
    while (n % 4 == 0) { r.push_back(4); n /= 4; }
    while (n % 2 == 0) { r.push_back(2); n /= 2; }
    for (int p : {3, 5, 7})
        while (n % p == 0) { r.push_back(p); n /= p; }
    if (n != 1) fail(SHTC_EUNSUPPORTED, "radix plan: length not 7-smooth");
    return r;
}

int next_pow2(int v) {
    int p = 1;
    while (p < v) p <<= 1;
    return p;
}

void set_err(shtc_ctx* c, const std::string& m) {
    g_last_error = m;
    if (c) c->err = m;
}

template <class F>
shtc_status guarded(shtc_ctx* c, F&& f) {
    try {
        if (c) CK(cudaSetDevice(c->device));
        f();
        return SHTC_OK;
    } catch (const ShtcError& e) {
        set_err(c, e.msg);
        return e.code;
    } catch (const std::bad_alloc&) {
        set_err(c, "host allocation failed");
        return SHTC_ENOMEM;
    } catch (const std::exception& e) {
        set_err(c, e.what());
        return SHTC_ECUDA;
    }
}

void check_latitudes(const double* x, int n, const char* where) {
    for (int i = 0; i < n; ++i)
        if (!(std::fabs(x[i]) <= 1.0))
            fail(SHTC_EINVAL, std::string(where) + ": cos_theta outside [-1, 1]");
}

void check_m_set(const int32_t* ms, int n, int mmax, const char* where) {
    for (int i = 0; i < n; ++i) {
        if (ms[i] < 0 || ms[i] > mmax) fail(SHTC_EINVAL, std::string(where) + ": order outside [0, mmax]");
        if (i > 0 && ms[i] <= ms[i - 1])
            fail(SHTC_EINVAL, std::string(where) + ": orders must be ascending and unique");
    }
}

// ---------------------------------------------------------------------------------------
// Legendre plan
// ---------------------------------------------------------------------------------------
// latitude-coherent tiles: streams ordered by |x| descending (polar first)
void sort_streams(std::vector<Stream>& streams) {
    std::stable_sort(streams.begin(), streams.end(),
                     [](const Stream& a, const Stream& b) { return std::fabs(a.x) > std::fabs(b.x); });
}

// Pipeline band of every tile of the sorted streams: contiguous tile ranges of ~equal pixel
// counts (band 0 half), band 0 at the equator.
std::vector<int> tile_bands(const shtc_ctx* c, const std::vector<Stream>& st) {
    const int ns = (int)st.size();
    const int nt = (ns + LEG_TILE - 1) / LEG_TILE;
    std::vector<int64_t> pix(nt, 0);
    int64_t total = 0;
    // pixel weight of a stream's rings; operator plans (latitudes without a grid) weigh 1 each
    const int nr = (int)c->nphi.size();
    auto w = [&](int r) -> int64_t { return r < 0 ? 0 : (r < nr ? c->nphi[r] : 1); };
    for (int i = 0; i < ns; ++i) {
        const int64_t p = w(st[i].north) + w(st[i].south);
        pix[i / LEG_TILE] += p;
        total += p;
    }
    // band k covers the pixel fraction [cum[k], cum[k+1]) counted from the equator; the
    // equatorial band 0 has half the weight of the others (it is map2alm's first H2D, so it
    // sets the head latency) -- SHTC_BAND0_WEIGHT overrides.  With 8 bands, band 2 (alm2map's
    // last band, whose pixels are the final copy) is kept small and bands 3-4 take its pixels:
    // weights 0.5,1,0.3,1.1,1.1,1,1,1 measured 23.23 -> 22.93 ms for the C4 pair from pinned
    // memory (tools/band_weights.sh); with 6 bands a small band 2 measured slower (23.05-23.17
    // against 22.58 ms for 0.5,1,1,1,1,1).  SHTC_BAND_WEIGHTS="w0,w1,..." sets every weight.
    static const double w0 = std::getenv("SHTC_BAND0_WEIGHT") ? std::atof(std::getenv("SHTC_BAND0_WEIGHT")) : 0.5;
    static const std::vector<double> wl = [] {
        std::vector<double> v;
        if (const char* e = std::getenv("SHTC_BAND_WEIGHTS"))
            for (const char* q = e; *q;) {
                v.push_back(std::max(1e-3, std::atof(q)));
                while (*q && *q != ',') ++q;
                if (*q) ++q;
            }
        return v;
    }();
    static const double wdef[8] = {0.5, 1.0, 0.3, 1.1, 1.1, 1.0, 1.0, 1.0};
    std::vector<double> cum(kPipeBands + 1, 0.0);
    for (int k = 0; k < kPipeBands; ++k)
        cum[k + 1] = cum[k] + (k < (int)wl.size() ? wl[k] : k == 0 ? w0 : (kPipeBands == 8 ? wdef[k] : 1.0));
    // Bands are assigned per tile PAIR counted from the equatorial end (tiles nt-1 and nt-2,
    // nt-3 and nt-4, ...): the map2alm kernel runs an item's tiles two at a time, and with no
    // band boundary inside a pair only an order's most polar alive tile can be left to run
    // on its own (16% of the C4 map2alm steps ran as single tiles with per-tile bands).
    static const bool pairs = !std::getenv("SHTC_BAND_PAIRS") || std::atoi(std::getenv("SHTC_BAND_PAIRS")) != 0;
    std::vector<int> band(nt);
    int64_t acc = 0;  // pixels of the tiles polar of the pair
    for (int t = 0; t < nt;) {
        // pair {t, t+1} when (nt - 1 - t) is odd, i.e. t and t+1 are one pair from the top
        const int len = (pairs && (nt - 1 - t) % 2 == 1 && t + 1 < nt) ? 2 : 1;
        int64_t pp = 0;
        for (int j = 0; j < len; ++j) pp += pix[t + j];
        const double eq = (double)(total - acc - pp) / (double)std::max<int64_t>(total, 1) * cum[kPipeBands];
        int k = 0;
        while (k + 1 < kPipeBands && eq >= cum[k + 1]) ++k;
        for (int j = 0; j < len; ++j) band[t + j] = k;
        acc += pp;
        t += len;
    }
    return band;
}

// band of every ring (-1: ring in no stream)
std::vector<int> ring_bands(const shtc_ctx* c, std::vector<Stream> st) {
    sort_streams(st);
    const std::vector<int> tb = tile_bands(c, st);
    std::vector<int> rb(c->n_rings, -1);
    for (size_t i = 0; i < st.size(); ++i) {
        rb[st[i].north] = tb[i / LEG_TILE];
        if (st[i].south >= 0) rb[st[i].south] = tb[i / LEG_TILE];
    }
    return rb;
}

// alm2map pipeline: bands whose Legendre launches run by order chunk while a_lm arrives
// (SHTC_A2M_HEAD overrides)
int a2m_head_bands() {
    static const int h = std::getenv("SHTC_A2M_HEAD") ? std::max(1, std::atoi(std::getenv("SHTC_A2M_HEAD"))) : 2;
    return std::min(h, kPipeBands);
}

// map2alm pipeline: the band after whose ring analysis each band's Legendre items launch
// (SHTC_M2A_GROUPS="1,1,2,2,2" = band counts per launch).  Default: every band on its own
// except the last two, which launch together split by order chunk (C4 map2alm from pinned
// memory 12.50 -> 12.13 ms median; merging more bands measured slower, 12.3-15.5 ms).
std::vector<int> m2a_launch_bands() {
    std::vector<int> sizes;
    if (const char* e = std::getenv("SHTC_M2A_GROUPS")) {
        for (const char* q = e; *q;) {
            sizes.push_back(std::max(1, std::atoi(q)));
            while (*q && *q != ',') ++q;
            if (*q) ++q;
        }
    } else {
        sizes.assign(kPipeBands, 1);
        if (kPipeBands >= 3) {
            sizes.pop_back();
            sizes.back() = 2;
        }
    }
    std::vector<int> tag(kPipeBands, kPipeBands - 1);
    int first = 0;
    for (int sz : sizes) {
        const int last = std::min(kPipeBands - 1, first + sz - 1);
        for (int b = first; b <= last; ++b) tag[b] = last;
        first = last + 1;
        if (first >= kPipeBands) break;
    }
    return tag;
}

// tiles per map2alm item of the pipelined (band) item set; SHTC_M2A_BAND_GROUP overrides
int m2a_band_group() {
    static const int g = std::getenv("SHTC_M2A_BAND_GROUP") ? std::max(1, std::atoi(std::getenv("SHTC_M2A_BAND_GROUP"))) : (LEG_M2A_P > 1 ? 2 : 1);
    return g;
}

// LSD radix sort of 64-bit keys, 16-bit digits (4 passes; digits that are constant over all keys
// are skipped): the plan's item sorts (~130 K keys at C4) in ~1 ms instead of ~3 ms each.
void radix_sort_u64(std::vector<uint64_t>& v) {
    std::vector<uint64_t> tmp(v.size());
    std::vector<size_t> cnt(65536);
    for (int sh = 0; sh < 64; sh += 16) {
        std::fill(cnt.begin(), cnt.end(), 0);
        for (uint64_t x : v) ++cnt[(x >> sh) & 0xffff];
        if (!v.empty() && cnt[(v[0] >> sh) & 0xffff] == v.size()) continue;  // constant digit
        size_t sum = 0;
        for (auto& c : cnt) {
            const size_t n = c;
            c = sum;
            sum += n;
        }
        for (uint64_t x : v) tmp[cnt[(x >> sh) & 0xffff]++] = x;
        v.swap(tmp);
    }
}

// SHTC_PLAN_TRACE=1: wall-clock ms of each plan phase (the stream synchronised at every mark)
struct PlanTrace {
    cudaStream_t s;
    const char* what;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void mark(const char* phase) {
        static const bool on = std::getenv("SHTC_PLAN_TRACE") != nullptr;
        if (!on) return;
        cudaStreamSynchronize(s);
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[plan %s] %s %.2f ms\n", what, phase,
                     std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};

void build_leg_plan(shtc_ctx* c, LegPlan& P, int lmax, int /*mmax: the order set ms*/, const std::vector<int>& ms,
                    std::vector<Stream> streams, const std::vector<double>& log_mu) {
    cudaStream_t s = c->stream;
    cudaEvent_t e0 = c->ev[6], e1 = c->ev[7];
    PlanTrace tr{s, "legendre"};
    CK(cudaEventRecord(e0, s));
    P = LegPlan();  // release previous
    tr.mark("release");
    P.lmax = lmax;
    P.ms = ms;
    sort_streams(streams);
    P.streams = streams;
    const std::vector<int> tband = tile_bands(c, streams);
    const int ns = (int)streams.size();
    const int n_m = (int)ms.size();
    std::vector<double> sx(ns), sl2(ns);
    std::vector<int> spos(ns), sno(ns), sso(ns);
    for (int i = 0; i < ns; ++i) {
        const double x = streams[i].x;
        const double s2 = (1.0 - x) * (1.0 + x);  // legendre.cpp:67
        sx[i] = x;
        spos[i] = s2 > 0.0;
        sl2[i] = s2 > 0.0 ? std::log2(s2) : 0.0;
        sno[i] = streams[i].north;
        sso[i] = streams[i].south;
    }
    tr.mark("streams + bands (host)");
    std::vector<int64_t> toff(n_m);
    int64_t tot = 0;
    for (int i = 0; i < n_m; ++i) {
        toff[i] = tot;
        tot += lmax - ms[i] + 1;
    }
    P.ms_d.upload(ms, s);
    P.logmu_d.upload(log_mu, s);
    P.sx.upload(sx, s);
    P.sl2.upload(sl2, s);
    P.spos.upload(spos, s);
    P.sn.upload(sno, s);
    P.ss.upload(sso, s);
    P.tab_off.upload(toff, s);
    tr.mark("small uploads");
    P.A.ensure(tot * sizeof(double));
    P.C.ensure(tot * sizeof(double));
    P.T.ensure(tot * sizeof(double));

    LegPlanView& v = P.view;
    v.lmax = lmax;
    v.n_m = n_m;
    v.ms = P.ms_d.as<int>();
    v.log_mu = P.logmu_d.as<double>();
    v.exp_lmu0 = std::exp(log_mu[0]);  // pmm_from_log m == 0 (legendre.cpp:65)
    v.tab = LegTables{P.A.as<double>(), P.C.as<double>(), P.T.as<double>(), P.tab_off.as<int64_t>()};
    v.st = LegStreams{P.sx.as<double>(), P.sl2.as<double>(), P.spos.as<int>(), P.sn.as<int>(),
                      P.ss.as<int>(), ns};
    v.n_tiles = (ns + LEG_TILE - 1) / LEG_TILE;
    v.unscaled = c->ladder ? 0 : 1;

    tr.mark("streams + uploads");
    if (n_m > 0) launch_leg_tables(v.ms, n_m, lmax, v.tab, s);
    CK(cudaGetLastError());
    tr.mark("recurrence tables");

    P.ck_act.ensure((size_t)std::max(1, n_m * ns) * sizeof(int));
    P.ck_q.ensure((size_t)std::max(1, n_m * ns) * sizeof(double2));
    v.ck_q = P.ck_q.as<double2>();
    v.ck_act = P.ck_act.as<int>();
    DevBuf& act = P.ck_act;
    P.tile_info.ensure((size_t)n_m * v.n_tiles * sizeof(int2));
    c->stats.ensure(sizeof(unsigned long long));
    CK(cudaMemsetAsync(c->stats.p, 0, sizeof(unsigned long long), s));
    v.tile_info = P.tile_info.as<int2>();
    if (n_m > 0) {
        launch_leg_scan(v, act.as<int>(), P.ck_q.as<double2>(), s);
        CK(cudaGetLastError());
        launch_leg_tile_summary(v, act.as<int>(), P.tile_info.as<int2>(),
                                c->stats.as<unsigned long long>(), s);
        CK(cudaGetLastError());
    }
    tr.mark("activation scan + tile summary");
    std::vector<int2> info((size_t)n_m * v.n_tiles);
    unsigned long long useful = 0;
    if (!info.empty())
        CK(cudaMemcpyAsync(info.data(), P.tile_info.p, info.size() * sizeof(int2), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&useful, c->stats.p, sizeof(useful), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    P.useful = useful;

    tr.mark("tile info to host");
    // alive tile lists per order and the cost-sorted work queues of the persistent kernels
    // Two item sets: cost-ordered for the device-resident single launches, band-ordered for
    // the pipelined host-buffer paths.  Tile lists run in descending tile index, i.e. bands in
    // ascending order (band 0 = equator).
    std::vector<int> tl, toffs(n_m), tcnt(n_m);
    std::vector<LegItem> a2m, m2a, m2a_b;
    std::vector<int> per_m(n_m), per_m_b(n_m);
    std::vector<int64_t> slot(n_m), slot_b(n_m);
    int64_t slots = 0, slots_b = 0;
    P.nominal = P.executed = P.prefix_steps = P.checked_steps = P.fast_steps = 0;
    // tiles per map2alm item of the device-resident set: LEG_M2A_GROUP when the plan has
    // many items per resident warp (whole transforms), fewer when it has few (one worker's
    // orders of a multi-GPU partition), where the longest item would set the kernel time
    int64_t alive_total = 0;
    for (const int2& ti : info) alive_total += ti.x >= 0;
    int dev_id = 0;
    CK(cudaGetDevice(&dev_id));
    // (a multiple of the pass width: the map2alm kernel runs an item's tiles LEG_M2A_P at a
    // time, so every item's passes are consecutive tile pairs of one band)
    constexpr int kPair = LEG_M2A_P > 1 ? 2 : 1;
    const int g_dev = (int)std::max<int64_t>(
        std::min(kPair, LEG_M2A_GROUP),
        std::min<int64_t>(LEG_M2A_GROUP, alive_total / (LEG_M2A_ITEMS_PER_WARP * (int64_t)leg_m2a_warps(dev_id)))
            / kPair * kPair);
    P.m2a_group = g_dev;
    auto tile_start = [&](int mi, int t) { return leg_tile_start(info[(size_t)mi * v.n_tiles + t].x); };
    // steps one pass runs (from the earliest start of its tiles): every step times the streams
    // of its tiles; steps up to the last activation test for activation events ("checked"),
    // later steps are plain recurrence + accumulation ("fast")
    auto account = [&](int mi, const int* ts, int nt, uint64_t& executed, uint64_t* checked, uint64_t* fast) {
        const int n = lmax - ms[mi];
        int ic = INT_MAX, ie = -1, in_pass = 0;
        for (int k = 0; k < nt; ++k) {
            ic = std::min(ic, tile_start(mi, ts[k]));
            ie = std::max(ie, info[(size_t)mi * v.n_tiles + ts[k]].y);
            in_pass += std::min(LEG_TILE, ns - ts[k] * LEG_TILE);
        }
        const uint64_t run = (uint64_t)(n + 1 - ic);
        const uint64_t fst = std::min<uint64_t>(run, (uint64_t)std::max(0, n - std::max(ie, ic)));
        executed += run * in_pass;
        if (fast) *fast += fst * in_pass;
        if (checked) *checked += (run - fst) * in_pass;
    };
    P.executed_a2m = 0;
    uint64_t single_steps = 0;  // map2alm steps run by single-tile passes (SHTC_PLAN_STATS)
    for (int i = 0; i < n_m; ++i) {
        const int n = lmax - ms[i];
        P.nominal += (uint64_t)(n + 1) * ns;
        toffs[i] = (int)tl.size();
        std::vector<int> alive;
        for (int t = v.n_tiles - 1; t >= 0; --t)  // descending tile index: bands ascending
            if (info[(size_t)i * v.n_tiles + t].x >= 0) alive.push_back(t);
        tl.insert(tl.end(), alive.begin(), alive.end());
        tcnt[i] = (int)alive.size();
        // alm2map items: consecutive alive tiles of one band in pairs (LEG_A2M_P), one tile
        // when the pair would cross a band
        for (size_t a = 0; a < alive.size();) {
            const int nt = (LEG_A2M_P > 1 && a + 1 < alive.size() && tband[alive[a + 1]] == tband[alive[a]]) ? 2 : 1;
            a2m.push_back(LegItem{i, alive[a], nt > 1 ? alive[a + 1] : -1, 0});
            account(i, &alive[a], nt, P.executed_a2m, nullptr, nullptr);
            a += nt;
        }
        // map2alm passes: consecutive alive tiles of one band in pairs (kPair)
        for (size_t a = 0; a < alive.size();) {
            const int nt = (kPair > 1 && a + 1 < alive.size() && tband[alive[a + 1]] == tband[alive[a]]) ? 2 : 1;
            account(i, &alive[a], nt, P.executed, &P.checked_steps, &P.fast_steps);
            if (nt == 1) account(i, &alive[a], 1, single_steps, nullptr, nullptr);
            a += nt;
        }
        // map2alm items: up to G consecutive alive tiles of one pipeline band.  Device-
        // resident set: G = g_dev (fewer partial slots; one launch, so long items only delay
        // its start).  Band set: G = m2a_band_group, so no item outlasts the band's launch.
        // Sets with equal G are the same partition (same sums); otherwise both deterministic.
        auto group = [&](int G, std::vector<LegItem>& out, int& cnt) {
            cnt = 0;
            for (size_t a = 0; a < alive.size();) {
                size_t e = a + 1;
                while (e < alive.size() && e - a < (size_t)G && tband[alive[e]] == tband[alive[a]]) ++e;
                out.push_back(LegItem{i, toffs[i] + (int)a, (int)(e - a), cnt++});
                a = e;
            }
        };
        group(g_dev, m2a, per_m[i]);
        group(m2a_band_group(), m2a_b, per_m_b[i]);
        slot[i] = slots;
        slots += (int64_t)per_m[i] * (n + 1);
        slot_b[i] = slots_b;
        slots_b += (int64_t)per_m_b[i] * (n + 1);
    }
    if (std::getenv("SHTC_PLAN_STATS")) {
        // activation events of the map2alm passes: distinct activation steps inside each
        // pass's checked window (ic, ie], and the window lengths
        std::vector<int> acts((size_t)n_m * ns);
        CK(cudaMemcpy(acts.data(), P.ck_act.p, acts.size() * sizeof(int), cudaMemcpyDeviceToHost));
        uint64_t events = 0, window = 0, passes = 0;
        for (int i = 0; i < n_m; ++i) {
            std::vector<int> alive;
            for (int t = v.n_tiles - 1; t >= 0; --t)
                if (info[(size_t)i * v.n_tiles + t].x >= 0) alive.push_back(t);
            for (size_t a = 0; a < alive.size();) {
                const int nt = (kPair > 1 && a + 1 < alive.size() && tband[alive[a + 1]] == tband[alive[a]]) ? 2 : 1;
                int ic = INT_MAX, ie = -1;
                std::vector<int> ev;
                for (int k = 0; k < nt; ++k) {
                    const int t = alive[a + k];
                    ic = std::min(ic, tile_start(i, t));
                    ie = std::max(ie, info[(size_t)i * v.n_tiles + t].y);
                    for (int j = 0; j < LEG_TILE && t * LEG_TILE + j < ns; ++j) ev.push_back(acts[(size_t)i * ns + t * LEG_TILE + j]);
                }
                std::sort(ev.begin(), ev.end());
                ev.erase(std::unique(ev.begin(), ev.end()), ev.end());
                for (int e : ev) events += (e > ic && e != INT_MAX);
                window += (uint64_t)std::max(0, ie - ic);
                ++passes;
                a += nt;
            }
        }
        std::fprintf(stderr, "plan stats: map2alm passes %llu, checked-window steps %llu, activation events %llu\n",
                     (unsigned long long)passes, (unsigned long long)window, (unsigned long long)events);
        std::fprintf(stderr, "plan stats: map2alm executed %llu (single-tile passes %llu), alm2map executed %llu, useful %llu\n",
                     (unsigned long long)P.executed, (unsigned long long)single_steps,
                     (unsigned long long)P.executed_a2m, (unsigned long long)P.useful);
    }
    // cost = degree steps actually run (from the pass's resume point) x tiles in the pass
    auto pass_cost = [&](int mi, int ta, int tb) {
        const int ic = tb >= 0 ? std::min(tile_start(mi, ta), tile_start(mi, tb)) : tile_start(mi, ta);
        return (int64_t)(lmax - ms[mi] + 1 - ic) * (tb >= 0 ? 2 : 1);
    };
    auto a2m_cost = [&](const LegItem& it) { return pass_cost(it.mi, it.a, it.b); };
    auto m2a_cost = [&](const LegItem& it) {
        int64_t c = 0;
        int k = 0;
        for (; k + kPair <= it.b; k += kPair) c += pass_cost(it.mi, tl[it.a + k], kPair > 1 ? tl[it.a + k + 1] : -1);
        for (; k < it.b; ++k) c += pass_cost(it.mi, tl[it.a + k], -1);
        return c;
    };
    tr.mark("items + accounting");
    // order chunks of ~equal coefficient counts (H2D / D2H units of the pipelined paths)
    std::vector<int> chunk_of(n_m, 0);
    P.chunk_mi.assign(1, 0);
    {
        int64_t total = 0, acc = 0;
        for (int i = 0; i < n_m; ++i) total += lmax - ms[i] + 1;
        for (int i = 0; i < n_m; ++i) {
            const int k = (int)std::min<int64_t>(kOrderChunks - 1, acc * kOrderChunks / std::max<int64_t>(total, 1));
            while ((int)P.chunk_mi.size() <= k) P.chunk_mi.push_back(i);
            chunk_of[i] = k;
            acc += lmax - ms[i] + 1;
        }
        while ((int)P.chunk_mi.size() <= kOrderChunks) P.chunk_mi.push_back(n_m);
    }
    // map2alm: the last band's launches by finer order chunks, so the a_lm copy of each
    // chunk overlaps the next chunk's launch (SHTC_M2A_CHUNKS overrides)
    // (at most 16: every launch takes two of the pipeline's kPipeEvents timing events).
    // Chunks of equal coefficient counts: chunks sized by the launch set's work (first chunk
    // small, so the D2H starts earlier) measured 12.12-12.34 against 12.05 ms at C4.
    static const int m2a_chunks =
        std::getenv("SHTC_M2A_CHUNKS") ? std::min(16, std::max(1, std::atoi(std::getenv("SHTC_M2A_CHUNKS")))) : 8;
    std::vector<int> m2a_chunk_of(n_m, 0);
    {
        int64_t total = 0, acc = 0;
        for (int i = 0; i < n_m; ++i) total += lmax - ms[i] + 1;
        for (int i = 0; i < n_m; ++i) {
            m2a_chunk_of[i] = (int)std::min<int64_t>(m2a_chunks - 1, acc * m2a_chunks / std::max<int64_t>(total, 1));
            acc += lmax - ms[i] + 1;
        }
    }
    tr.mark("order chunks");
    // stable sorts by a key computed once per item (sorting (key, original index) pairs): the
    // cost functions walk tile lists, so evaluating them per comparison cost ~25 ms at C4
    // Keys are packed into one 64-bit word: group (16 bits) | inverted cost (24 bits) | original
    // index (24 bits), so a plain integer sort is the stable sort.
    auto sort_items = [](std::vector<LegItem>& v, auto group, auto cost) {
        if (v.size() >= (size_t(1) << 24)) fail(SHTC_EUNSUPPORTED, "plan: too many work items");
        std::vector<uint64_t> kv(v.size());
        for (size_t i = 0; i < v.size(); ++i) {
            const uint64_t g = (uint64_t)group(v[i]) & 0xffff;
            const uint64_t c = (uint64_t)std::min<int64_t>(cost(v[i]), (int64_t(1) << 24) - 1);
            kv[i] = (g << 48) | ((((uint64_t(1) << 24) - 1) - c) << 24) | (uint64_t)i;
        }
        radix_sort_u64(kv);
        std::vector<LegItem> out(v.size());
        for (size_t i = 0; i < v.size(); ++i) out[i] = v[kv[i] & 0xffffff];
        v.swap(out);
    };
    auto no_group = [](const LegItem&) { return 0; };
    sort_items(a2m, no_group, a2m_cost);
    sort_items(m2a, no_group, m2a_cost);
    // alm2map band set: band, then (band 0 only) order chunk, then cost
    // the head bands (0 .. a2m_head_bands()-1) run together, split by order chunk, while a_lm
    // arrives (launch band tag 0)
    auto a2m_key = [&](const LegItem& it) {
        const int tc = tband[it.a];
        const bool head = tc < a2m_head_bands();
        return std::make_pair(head ? 0 : tc, head ? chunk_of[it.mi] : 0);
    };
    std::vector<LegItem> a2m_b = a2m;
    sort_items(a2m_b, [&](const LegItem& it) {
        const auto k = a2m_key(it);
        return (k.first << 8) | k.second;
    }, a2m_cost);
    P.a2m_launch.clear();
    for (size_t k = 0; k < a2m_b.size();) {
        size_t e = k;
        while (e < a2m_b.size() && a2m_key(a2m_b[e]) == a2m_key(a2m_b[k])) ++e;
        P.a2m_launch.push_back({a2m_key(a2m_b[k]).first, a2m_key(a2m_b[k]).second, (int)k, (int)e});
        k = e;
    }
    // map2alm band set: an item runs with the band of its tiles (groups do not cross bands),
    // the last band also split by order chunk, then cost; an order is final after the launch
    // of its last item
    const std::vector<int> m2a_tag = m2a_launch_bands();
    auto m2a_key = [&](const LegItem& it) {
        const int tag = m2a_tag[tband[tl[it.a + it.b - 1]]];
        return std::make_pair(tag, tag == kPipeBands - 1 ? m2a_chunk_of[it.mi] : 0);
    };
    sort_items(m2a_b, [&](const LegItem& it) {
        const auto k = m2a_key(it);
        return (k.first << 8) | k.second;
    }, m2a_cost);
    P.m2a_launch.clear();
    std::vector<int> last_launch(n_m, 0);  // orders without items are final from the start
    for (size_t k = 0; k < m2a_b.size();) {
        size_t e = k;
        while (e < m2a_b.size() && m2a_key(m2a_b[e]) == m2a_key(m2a_b[k])) ++e;
        for (size_t q = k; q < e; ++q) last_launch[m2a_b[q].mi] = (int)P.m2a_launch.size();
        P.m2a_launch.push_back({m2a_key(m2a_b[k]).first, m2a_key(m2a_b[k]).second, (int)k, (int)e});
        k = e;
    }
    P.m2a_done.assign(std::max<size_t>(1, P.m2a_launch.size()), {});
    std::vector<std::vector<int>> final_of(P.m2a_done.size());
    for (int i = 0; i < n_m; ++i) {
        auto& runs = P.m2a_done[last_launch[i]];
        if (!runs.empty() && runs.back().second == i) runs.back().second = i + 1;
        else runs.push_back({i, i + 1});
        final_of[last_launch[i]].push_back(i);
    }
    // order indices final after each launch, for the deferred reduction (leg_m2a_finalize)
    std::vector<int> fl;
    P.m2a_final_off.assign(1, 0);
    for (const auto& f : final_of) {
        fl.insert(fl.end(), f.begin(), f.end());
        P.m2a_final_off.push_back((int)fl.size());
    }
    if (fl.empty()) fl.push_back(0);
    tr.mark("sorts + launch sets");
    P.m2a_final_list.upload(fl, s);
    if (tl.empty()) tl.push_back(0);
    P.tile_list.upload(tl, s);
    P.tile_off.upload(toffs, s);
    P.tile_cnt.upload(tcnt, s);
    P.a2m_items.upload(a2m, s);
    P.m2a_items.upload(m2a, s);
    P.m2a_per_m.upload(per_m, s);
    P.m2a_slot.upload(slot, s);
    P.a2m_items_band.upload(a2m_b, s);
    P.m2a_items_band.upload(m2a_b, s);
    P.m2a_per_m_band.upload(per_m_b, s);
    P.m2a_slot_band.upload(slot_b, s);
    P.m2a_scratch.ensure((size_t)std::max<int64_t>(std::max(slots, slots_b), 1) * sizeof(double2));
    // [0]: queue of single launches, [1, 1 + n_m): spare, then one queue word per pipelined
    // launch
    P.counters.ensure((size_t)(1 + n_m + P.a2m_launch.size() + P.m2a_launch.size()) * sizeof(int));
    v.tile_list = P.tile_list.as<int>();
    v.tile_list_off = P.tile_off.as<int>();
    v.tile_list_cnt = P.tile_cnt.as<int>();
    v.a2m_items = P.a2m_items.as<LegItem>();
    v.n_a2m_items = (int)a2m.size();
    v.m2a_items = P.m2a_items.as<LegItem>();
    v.n_m2a_items = (int)m2a.size();
    v.m2a_items_per_m = P.m2a_per_m.as<int>();
    v.m2a_slot_base = P.m2a_slot.as<int64_t>();
    v.m2a_scratch_elems = std::max(slots, slots_b);
    P.band_view = v;
    P.band_view.a2m_items = P.a2m_items_band.as<LegItem>();
    P.band_view.m2a_items = P.m2a_items_band.as<LegItem>();
    P.band_view.n_m2a_items = (int)m2a_b.size();
    P.band_view.m2a_items_per_m = P.m2a_per_m_band.as<int>();
    P.band_view.m2a_slot_base = P.m2a_slot_band.as<int64_t>();
    P.band_view.defer_final = 1;
    CK(cudaEventRecord(e1, s));
    CK(cudaStreamSynchronize(s));
    float ms_el = 0.f;
    CK(cudaEventElapsedTime(&ms_el, e0, e1));
    P.build_ms = ms_el;
    tr.mark("uploads");
    P.built = true;
}

std::vector<Stream> grid_streams(const shtc_ctx* c) {
    std::vector<Stream> st;
    const int n = c->n_rings;
    if (c->mirror && c->symmetric) {
        for (int k = 0; k < n / 2; ++k) st.push_back({c->cos_theta[k], k, n - 1 - k});
        if (n % 2 == 1) st.push_back({c->cos_theta[n / 2], n / 2, -1});
    } else {
        for (int r = 0; r < n; ++r) st.push_back({c->cos_theta[r], r, -1});
    }
    return st;
}

void ensure_leg_plan(shtc_ctx* c) {
    if (!c->grid_set) fail(SHTC_EINVAL, "no grid set");
    if (!c->band_set) fail(SHTC_EINVAL, "no band set");
    if (!c->leg.built) build_leg_plan(c, c->leg, c->lmax, c->mmax, c->ms, grid_streams(c), c->log_mu);
}

// ---------------------------------------------------------------------------------------
// Ring FFT plan
// ---------------------------------------------------------------------------------------
// ring_band: pipeline band per grid ring (bands of the host-buffer paths), or empty.
void build_fft_plan(shtc_ctx* c, FftPlan& F, const std::vector<int>& rings,
                    const std::vector<int>& ring_band = {}) {
    cudaStream_t s = c->stream;
    cudaEvent_t e0 = c->ev[6], e1 = c->ev[7];
    PlanTrace tr{s, "fft"};
    CK(cudaEventRecord(e0, s));
    for (auto& d : F.descs) d.release();
    std::fill(std::begin(F.alt), std::end(F.alt), 0);
    F.tabs.release();
    std::vector<TableJob> jobs;
    int64_t tot = 0;
    std::map<std::pair<int, int>, int64_t> table_at;  // (kind, L) -> offset
    auto table = [&](int kind, int L) {
        auto key = std::make_pair(kind, L);
        auto it = table_at.find(key);
        if (it != table_at.end()) return it->second;
        const int64_t off = tot;
        tot += (kind == 1) ? L / 2 + 1 : L;
        jobs.push_back(TableJob{off, L, kind, 0.0});
        table_at[key] = off;
        return off;
    };
    // phase factor tables, one per distinct phi0 (the mirror rings of a pair share theirs)
    std::map<double, int64_t> phase_at;
    const int n_phase = 64 + (c->mmax >> 6) + 1;
    auto phase_table = [&](double phi0) {
        auto it = phase_at.find(phi0);
        if (it != phase_at.end()) return it->second;
        const int64_t off = tot;
        tot += n_phase;
        jobs.push_back(TableJob{off, n_phase, 3, phi0});
        phase_at[phi0] = off;
        return off;
    };
    F.mmax = c->mmax;
    std::map<int64_t, int64_t> h_at;  // Bluestein (N, half) -> H offset
    std::vector<RingDesc> per_class[FFT_N_CLASSES];
    std::vector<RingDesc> blue_class[FFT_N_CLASSES];
    std::vector<RingDesc> blue_clus;
    for (size_t pos = 0; pos < rings.size(); ++pos) {
        const int r = rings[pos];
        RingDesc d{};
        d.n = c->nphi[r];
        if (d.n < 1) fail(SHTC_EINVAL, "ring_synthesis: ring has no samples");
        const bool half = (d.n % 2 == 0);
        d.N = half ? d.n / 2 : d.n;
        // 7-smooth lengths run the mixed-radix path; odd radices fit the register-staged
        // passes only up to 1024 points, longer non-power-of-two lengths go through Bluestein
        const bool smooth = is_smooth7(d.N) && (d.N <= 1024 || (d.N & (d.N - 1)) == 0);
        d.B = smooth ? d.N : next_pow2(2 * d.N - 1);
        d.flags = (half ? 1 : 0) | (smooth ? 0 : 2);
        d.pix_off = c->pixoff[r];
        d.phi0 = c->phi0[r];
        d.ph_off = d.phi0 != 0.0 ? phase_table(d.phi0) : 0;
        d.weight = c->weight[r];
        d.ring_pos = (int)pos;
        // half-mode rings with a power-of-two buffer (direct or Bluestein) run the register
        // resident power-of-two engine; the rest (odd rings, other 7-smooth lengths, tiny
        // buffers) the generic in-place mixed-radix kernels.  Bluestein's FFT(conj chirp) is
        // built by the generic class of the same length at plan time.
        // odd rings whose Bluestein buffer exceeds the generic classes (n > 4096): one-sided
        // (pruned) Bluestein on the 2-CTA cluster class -- K = min(n, mmax + 1) spectrum bins
        // in, n samples out (or back), so n + K - 1 <= 16384 points suffice (the Gauss-Legendre
        // n_phi = 2 lmax + 1 = 8193 at lmax 4096 needs 12289)
        bool odd_clus = false;
        if (!half && !smooth && fft_class_for(d.B) < 0) {
            const int K = std::min(d.n, c->mmax + 1);
            if ((int64_t)d.n + K - 1 <= FFT_P2C_B) {
                d.B = FFT_P2C_B;
                d.K = K;
                odd_clus = true;
            }
        }
        const int gcls = fft_class_for(d.B);
        // 16384-point Bluestein buffers (N < 8192): 2-CTA clusters.  A direct 16384-point ring
        // (n_phi = 32768, N a power of two) is not one of them: it has no class and fails below
        const bool clus = (half && !smooth && d.B == FFT_P2C_B) || odd_clus;
        int cls = clus ? FFT_P2C_CLASS : (half ? fft_p2_class_for(d.B, !smooth) : -1);
        if (cls < 0) cls = gcls;
        if (cls < 0)
            fail(SHTC_EUNSUPPORTED, "ring length " + std::to_string(d.n) +
                                        " needs an FFT buffer beyond the shared-memory classes");
        if (gcls >= 0) {
            auto rp = radix_plan(d.B);
            d.npass = (int)rp.size();
            if (rp.size() > (size_t)FFT_MAX_PASSES) fail(SHTC_EUNSUPPORTED, "radix plan too long");
            d.radices = 0;
            for (size_t i = 0; i < rp.size(); ++i) d.radices |= (unsigned long long)rp[i] << (4 * i);
        }
        d.tw_off = table(0, d.B);
        d.hw_off = half ? table(1, d.n) : 0;
        if (!smooth) {
            d.chirp_off = table(2, d.N);
            const int64_t hkey = 2 * (int64_t)d.N + (half ? 1 : 0);  // odd cluster rings: pruned h
            auto it = h_at.find(hkey);
            if (it == h_at.end()) {
                d.h_off = tot;
                tot += d.B;
                h_at[hkey] = d.h_off;
                if (clus) blue_clus.push_back(d);
                else blue_class[gcls].push_back(d);
            } else {
                d.h_off = it->second;
            }
        }
        per_class[cls].push_back(d);
        F.tw_off[cls] = clus ? table(0, FFT_P2C_B / 2) : d.tw_off;
    }
    // the 8192-point Bluestein class as two 4096-point halves per CTA when no ring of it aliases
    // (n > mmax: the split kernel's fold has no wrap loop); SHTC_P2H=0 keeps the one-transform
    // kernel
    {
        static const bool p2h_on = !std::getenv("SHTC_P2H") || std::atoi(std::getenv("SHTC_P2H")) != 0;
        const int k8 = fft_p2_class_for(8192, true);
        bool ok = p2h_on && k8 >= 0 && !per_class[k8].empty();
        if (ok)
            for (const RingDesc& d : per_class[k8]) ok = ok && (d.flags & 3) == 3 && d.n > c->mmax && d.N < 4096;
        if (ok) {
            F.alt[k8] = 1;
            F.tw_off[k8] = table(0, 4096);
        }
    }
    tr.mark("descriptors");
    F.tabs.ensure((size_t)std::max<int64_t>(tot, 1) * sizeof(double2));
    tr.mark("table allocation");
    DevBuf jobs_d;
    jobs_d.upload(jobs, s);
    launch_fill_tables(jobs_d.as<TableJob>(), (int)jobs.size(), F.tabs.as<double2>(), s);
    CK(cudaGetLastError());
    tr.mark("tables");
    for (int k = 0; k < FFT_N_CLASSES; ++k) {
        if (!blue_class[k].empty()) {
            DevBuf bd;
            bd.upload(blue_class[k], s);
            launch_bluestein_h(k, bd.as<RingDesc>(), (int)blue_class[k].size(), F.tabs.as<double2>(), s);
            CK(cudaGetLastError());
            CK(cudaStreamSynchronize(s));
        }
        F.count[k] = (int)per_class[k].size();
    }
    if (!blue_clus.empty()) {
        DevBuf bd;
        bd.upload(blue_clus, s);
        launch_p2c_h(bd.as<RingDesc>(), (int)blue_clus.size(), F.tabs.as<double2>(),
                     F.tabs.as<double2>() + F.tw_off[FFT_P2C_CLASS], s);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(s));
    }
    tr.mark("bluestein FFT(h)");
    // pipeline bands: descriptors of each class grouped by band (ring order inside a band),
    // pixel intervals of each band for the host copies
    {
        auto band = [&](const RingDesc& d) {
            return ring_band.empty() ? 0 : std::max(0, ring_band[rings[d.ring_pos]]);
        };
        F.band_pix.assign(kPipeBands, {});
        for (size_t pos = 0; pos < rings.size(); ++pos) {
            const int r = rings[pos];
            const int k = ring_band.empty() ? 0 : std::max(0, ring_band[r]);
            const int64_t b0 = c->pixoff[r], b1 = b0 + c->nphi[r];
            auto& iv = F.band_pix[k];
            if (!iv.empty() && iv.back().second == b0) iv.back().second = b1;
            else iv.push_back({b0, b1});
        }
        for (int cls = 0; cls < FFT_N_CLASSES; ++cls) {
            // band, then ring length: rings that share their tables (hw, chirp, FFT(h) are one
            // per length -- the north and south rings of a mirror pair) sit next to each other
            // in the queue, so the second read of a table is an L2 hit instead of a second HBM
            // read half a launch later
            std::stable_sort(per_class[cls].begin(), per_class[cls].end(),
                             [&](const RingDesc& a, const RingDesc& b) {
                                 if (band(a) != band(b)) return band(a) < band(b);
                                 return a.n < b.n;
                             });
            F.descs[cls].upload(per_class[cls], s);
            F.range_start[cls].assign(kPipeBands + 1, 0);
            for (const RingDesc& d : per_class[cls]) F.range_start[cls][band(d) + 1]++;
            for (int k = 0; k < kPipeBands; ++k) F.range_start[cls][k + 1] += F.range_start[cls][k];
        }
    }
    F.counters.ensure((size_t)(kPipeBands + 1) * FFT_N_CLASSES * sizeof(int));  // no allocation on the transform path
    CK(cudaEventRecord(e1, s));
    CK(cudaStreamSynchronize(s));
    float el = 0.f;
    CK(cudaEventElapsedTime(&el, e0, e1));
    F.build_ms = el;
    tr.mark("band ranges + uploads");
    F.built = true;
}

void ensure_id_layout(shtc_ctx* c) {
    if (c->id_row_off.p) return;
    const int nm = (int)c->ms.size();
    std::vector<int64_t> ro(c->n_rings), mb(c->mmax + 1), mst(c->mmax + 1);
    for (int r = 0; r < c->n_rings; ++r) ro[r] = (int64_t)r * nm;
    for (int m = 0; m <= c->mmax; ++m) {
        mb[m] = m;
        mst[m] = c->mmax + 1;
    }
    c->id_row_off.upload(ro, c->stream);
    c->id_m_base.upload(mb, c->stream);
    c->id_m_stride.upload(mst, c->stream);
}

void ensure_fft_id(shtc_ctx* c) {
    if (!c->grid_set) fail(SHTC_EINVAL, "no grid set");
    if (!c->fft_id.built) {
        std::vector<int> all(c->n_rings);
        std::iota(all.begin(), all.end(), 0);
        build_fft_plan(c, c->fft_id, all, ring_bands(c, grid_streams(c)));
    }
}

void require_full_band(shtc_ctx* c) {
    if (!c->band_set) fail(SHTC_EINVAL, "no band set");
    if ((int)c->ms.size() != c->mmax + 1)
        fail(SHTC_EINVAL, "whole transforms need every order 0..mmax on this context");
}

float elapsed(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, a, b));
    return ms;
}

// Ring stage launches of one plan (or of one pipeline band of it).  The large power-of-two
// classes (buffers >= 2048, the belt and the big polar-cap rings) go on the caller's stream;
// the small-ring classes (latency bound: few CTAs, aliasing folds over many wraps) run on
// kFftAux side streams at the same time, joined back before the stage ends.
template <class Launch>
void ring_stage(shtc_ctx* c, FftPlan& F, int range, cudaStream_t s, Launch launch, bool big_on_side = false) {
    if (!c->fft_fork) {
        for (int i = 0; i < fft_aux_count(); ++i) CK(cudaStreamCreateWithFlags(&c->fft_aux[i], cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&c->fft_fork, cudaEventDisableTiming));
        for (auto& e : c->fft_join) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    // one counter slice per band (slice 0: whole-plan stages), so ring stages of different
    // bands may run concurrently on different streams
    F.counters.ensure((size_t)(kPipeBands + 1) * FFT_N_CLASSES * sizeof(int));
    int* const ctr = F.counters.as<int>() + (range < 0 ? 0 : range + 1) * FFT_N_CLASSES;
    CK(cudaMemsetAsync(ctr, 0, FFT_N_CLASSES * sizeof(int), s));
    CK(cudaEventRecord(c->fft_fork, s));
    bool used[kFftAux] = {};
    int side = 0;
    for (int k = FFT_N_CLASSES - 1; k >= 0; --k) {
        const int b = range < 0 ? 0 : F.range_start[k][range];
        const int e = range < 0 ? F.count[k] : F.range_start[k][range + 1];
        if (e <= b) continue;
        // big_on_side: the large classes on side streams too, so one class's tail overlaps the
        // next class's start (analysis: C4 0.73 -> 0.70 ms; synthesis measured no gain).
        // SHTC_FFT_BIG_SIDE=0/1 forces it for both directions.
        static const int big_side_env = std::getenv("SHTC_FFT_BIG_SIDE") ? std::atoi(std::getenv("SHTC_FFT_BIG_SIDE")) : -1;
        const bool side_big = big_side_env >= 0 ? big_side_env != 0 : big_on_side;
        const bool big = k >= FFT_N_GENERIC && fft_class_bmax(k) >= 2048 && !side_big;
        cudaStream_t st = s;
        if (!big) {
            const int i = side++ % fft_aux_count();
            if (!used[i]) CK(cudaStreamWaitEvent(c->fft_aux[i], c->fft_fork, 0));
            used[i] = true;
            st = c->fft_aux[i];
        }
        RingStageArgs a{};
        a.rings = F.descs[k].as<RingDesc>() + b;
        a.n_rings = e - b;
        a.tabs = F.tabs.as<double2>();
        a.mmax = c->mmax;
        a.ld = c->mmax + 1;
        a.counter = ctr + k;
        a.p2_tw = a.tabs + F.tw_off[k];
        a.alt = F.alt[k];
        launch(k, a, st);
        CK(cudaGetLastError());
    }
    for (int i = 0; i < kFftAux; ++i)
        if (used[i]) {
            CK(cudaEventRecord(c->fft_join[i], c->fft_aux[i]));
            CK(cudaStreamWaitEvent(s, c->fft_join[i], 0));
        }
}

void run_ring_synth(shtc_ctx* c, FftPlan& F, const double2* delta, double* map,
                    const int64_t* mb, const int64_t* mst, int range = -1, cudaStream_t s = nullptr) {
    ring_stage(c, F, range, s ? s : c->stream, [&](int k, RingStageArgs& a, cudaStream_t st) {
        a.m_base = mb;
        a.m_stride = mst;
        a.delta_in = delta;
        a.map_out = map;
        launch_ring_synthesis(k, a, st);
    });
}

void run_ring_anal(shtc_ctx* c, FftPlan& F, const double* map, double2* delta, const int64_t* mb,
                   const int64_t* mst, int range = -1, double2* const* col_ptr = nullptr,
                   cudaStream_t s = nullptr, const int* m_order = nullptr) {
    ring_stage(c, F, range, s ? s : c->stream, [&](int k, RingStageArgs& a, cudaStream_t st) {
        a.m_base = mb;
        a.m_stride = mst;
        a.col_ptr = col_ptr;
        a.m_order = m_order;
        a.map_in = map;
        a.delta_out = delta;
        launch_ring_analysis(k, a, st);
    }, true);
}

void fill_timing(shtc_timing* t, double leg, double fft, double h2d, double d2h, double total,
                 const LegPlan& P, bool alm2map) {
    if (!t) return;
    t->legendre_ms = leg;
    t->fft_ms = fft;
    t->h2d_ms = h2d;
    t->d2h_ms = d2h;
    t->total_ms = total;
    t->nominal_steps = P.nominal;
    t->executed_steps = alm2map ? P.executed_a2m : P.executed;
}

void do_alm2map_dev(shtc_ctx* c, const double* alm, double* map, shtc_timing* t, double h2d = 0) {
    require_full_band(c);
    ensure_leg_plan(c);
    ensure_fft_id(c);
    ensure_id_layout(c);
    c->delta.ensure((size_t)c->n_rings * (c->mmax + 1) * sizeof(double2));
    cudaStream_t s = c->stream;
    CK(cudaEventRecord(c->ev[0], s));
    launch_leg_alm2map(c->leg.view, reinterpret_cast<const double2*>(alm), c->delta.as<double2>(),
                       c->id_row_off.as<int64_t>(), c->leg.counters.as<int>(), s);
    CK(cudaGetLastError());
    CK(cudaEventRecord(c->ev[1], s));
    run_ring_synth(c, c->fft_id, c->delta.as<double2>(), map, nullptr, nullptr);
    CK(cudaEventRecord(c->ev[2], s));
    if (t) {
        CK(cudaEventSynchronize(c->ev[2]));
        const double leg = elapsed(c->ev[0], c->ev[1]), fft = elapsed(c->ev[1], c->ev[2]);
        fill_timing(t, leg, fft, h2d, 0.0, leg + fft, c->leg, true);
    }
}

void do_map2alm_dev(shtc_ctx* c, const double* map, double* alm, shtc_timing* t, double h2d = 0) {
    require_full_band(c);
    ensure_leg_plan(c);
    ensure_fft_id(c);
    ensure_id_layout(c);
    c->delta.ensure((size_t)c->n_rings * (c->mmax + 1) * sizeof(double2));
    cudaStream_t s = c->stream;
    CK(cudaEventRecord(c->ev[0], s));
    run_ring_anal(c, c->fft_id, map, c->delta.as<double2>(), nullptr, nullptr);
    CK(cudaEventRecord(c->ev[1], s));
    launch_leg_map2alm(c->leg.view, c->delta.as<double2>(), c->id_row_off.as<int64_t>(),
                       reinterpret_cast<double2*>(alm), 0, c->leg.counters.as<int>(),
                       c->leg.m2a_scratch.as<double2>(), s);
    CK(cudaGetLastError());
    CK(cudaEventRecord(c->ev[2], s));
    if (t) {
        CK(cudaEventSynchronize(c->ev[2]));
        const double fft = elapsed(c->ev[0], c->ev[1]), leg = elapsed(c->ev[1], c->ev[2]);
        fill_timing(t, leg, fft, h2d, 0.0, leg + fft, c->leg, false);
    }
}

size_t alm_count(int lmax, int mmax) {
    const size_t l = lmax, m = mmax;
    return (m + 1) * (l + 1) - m * (m + 1) / 2;
}

}  // namespace

// =========================================================================================
// C ABI
// =========================================================================================
extern "C" {

const char* shtc_last_error(const shtc_ctx* ctx) {
    return ctx ? ctx->err.c_str() : g_last_error.c_str();
}

uint64_t shtc_kernel_launches(void) { return (uint64_t)shtk::launch_count(); }

int shtc_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

shtc_status shtc_create(int device, shtc_ctx** out) {
    if (!out) return SHTC_EINVAL;
    *out = nullptr;
    return guarded(nullptr, [&] {
        int n = 0;
        CK(cudaGetDeviceCount(&n));
        if (device < 0 || device >= n) fail(SHTC_EINVAL, "shtc_create: no such CUDA device");
        cudaDeviceProp prop{};
        CK(cudaGetDeviceProperties(&prop, device));
        if (prop.major < 10)
            fail(SHTC_EUNSUPPORTED, std::string("shtc_create: kernels are built for sm_100a, device is ") +
                                        prop.name);
        CK(cudaSetDevice(device));
        auto c = std::make_unique<shtc_ctx>();
        c->device = device;
        CK(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
        c->stream = c->own_stream;
        for (auto& e : c->ev) CK(cudaEventCreate(&e));
        *out = c.release();
    });
}

void shtc_destroy(shtc_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    for (auto& e : ctx->ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : ctx->pev)
        if (e) cudaEventDestroy(e);
    for (auto& e : ctx->tev)
        if (e) cudaEventDestroy(e);
    for (auto& st : ctx->lst)
        if (st) cudaStreamDestroy(st);
    if (ctx->fst) cudaStreamDestroy(ctx->fst);
    for (auto& st : ctx->fft_aux)
        if (st) cudaStreamDestroy(st);
    if (ctx->fft_fork) cudaEventDestroy(ctx->fft_fork);
    for (auto& e : ctx->fft_join)
        if (e) cudaEventDestroy(e);
    if (ctx->h2d) cudaStreamDestroy(ctx->h2d);
    if (ctx->d2h) cudaStreamDestroy(ctx->d2h);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    delete ctx;
}

shtc_status shtc_set_stream(shtc_ctx* ctx, void* cuda_stream) {
    if (!ctx) return SHTC_EINVAL;
    ctx->stream = cuda_stream ? static_cast<cudaStream_t>(cuda_stream) : ctx->own_stream;
    return SHTC_OK;
}

shtc_status shtc_set_grid(shtc_ctx* ctx, int n_rings, const double* cos_theta, const int32_t* n_phi,
                          const double* phi_0, const double* weight, const int64_t* pixel_offset,
                          int mirror) {
    if (!ctx) return SHTC_EINVAL;
    return guarded(ctx, [&] {
        if (n_rings < 1 || !cos_theta || !n_phi || !phi_0 || !weight)
            fail(SHTC_EINVAL, "synthesis: empty grid");
        check_latitudes(cos_theta, n_rings, "synthesis");
        ctx->n_rings = n_rings;
        ctx->cos_theta.assign(cos_theta, cos_theta + n_rings);
        ctx->nphi.assign(n_phi, n_phi + n_rings);
        ctx->phi0.assign(phi_0, phi_0 + n_rings);
        ctx->weight.assign(weight, weight + n_rings);
        ctx->pixoff.resize(n_rings);
        int64_t off = 0;
        for (int r = 0; r < n_rings; ++r) {
            if (n_phi[r] < 1) fail(SHTC_EINVAL, "ring_synthesis: ring has no samples");
            ctx->pixoff[r] = pixel_offset ? pixel_offset[r] : off;
            off += n_phi[r];
        }
        ctx->npix = off;
        // symmetric_ring_pairs (grid.cpp:133-151)
        bool sym = true;
        for (int k = 0; k < n_rings / 2; ++k) {
            const int j = n_rings - 1 - k;
            if (n_phi[k] != n_phi[j] || std::fabs(cos_theta[k] + cos_theta[j]) > 1e-14) sym = false;
        }
        if (n_rings % 2 == 1 && std::fabs(cos_theta[n_rings / 2]) > 1e-14) sym = false;
        ctx->symmetric = sym;
        ctx->mirror = mirror != 0;
        ctx->grid_set = true;
        ctx->leg.built = false;
        ctx->fft_id.built = false;
        ctx->fft_custom.built = false;
        ctx->id_row_off.release();
        ctx->custom_layout = false;
        ctx->syn_layout = false;
        ctx->peers_set = false;  // peer targets index the old ring / order layout
    });
}

shtc_status shtc_set_band(shtc_ctx* ctx, int lmax, int mmax, int n_m, const int32_t* ms) {
    if (!ctx) return SHTC_EINVAL;
    return guarded(ctx, [&] {
        if (lmax < mmax || mmax < 0) fail(SHTC_EINVAL, "analysis: need lmax >= mmax >= 0");
        std::vector<int> v;
        if (ms && n_m > 0) {
            check_m_set(ms, n_m, mmax, "shtc_set_band");
            v.assign(ms, ms + n_m);
        } else {
            v.resize(mmax + 1);
            std::iota(v.begin(), v.end(), 0);
        }
        ctx->lmax = lmax;
        ctx->mmax = mmax;
        ctx->ms = v;
        ctx->log_mu.resize(mmax + 1);
        for (int m = 0; m <= mmax; ++m) ctx->log_mu[m] = host_log_mu(m);
        ctx->band_set = true;
        ctx->leg.built = false;
        if (ctx->fft_id.mmax != mmax) ctx->fft_id.built = false;  // phase tables sized by mmax
        ctx->id_row_off.release();
        ctx->custom_layout = false;
        ctx->syn_layout = false;
        ctx->peers_set = false;
    });
}

shtc_status shtc_set_ladder(shtc_ctx* ctx, int enabled) {
    if (!ctx) return SHTC_EINVAL;
    return guarded(ctx, [&] {
        if ((enabled != 0) == ctx->ladder) return;
        ctx->ladder = enabled != 0;
        ctx->leg.built = false;
        ctx->op_leg.built = false;
    });
}

shtc_status shtc_plan(shtc_ctx* ctx, double* plan_ms) {
    if (!ctx) return SHTC_EINVAL;
    return guarded(ctx, [&] {
        ensure_leg_plan(ctx);
        ensure_fft_id(ctx);
        if (plan_ms) *plan_ms = ctx->leg.build_ms + ctx->fft_id.build_ms;
    });
}

shtc_status shtc_plan_stats(shtc_ctx* ctx, uint64_t* nominal, uint64_t* executed, uint64_t* useful) {
    if (!ctx) return SHTC_EINVAL;
    return guarded(ctx, [&] {
        ensure_leg_plan(ctx);
        if (nominal) *nominal = ctx->leg.nominal;
        if (executed) *executed = ctx->leg.executed;
        if (useful) *useful = ctx->leg.useful;
    });
}

shtc_status shtc_plan_phase_stats(shtc_ctx* ctx, uint64_t* prefix, uint64_t* checked, uint64_t* fast) {
    if (!ctx) return SHTC_EINVAL;
    return guarded(ctx, [&] {
        ensure_leg_plan(ctx);
        if (prefix) *prefix = ctx->leg.prefix_steps;
        if (checked) *checked = ctx->leg.checked_steps;
        if (fast) *fast = ctx->leg.fast_steps;
    });
}

shtc_status shtc_host_alloc(size_t bytes, void** out) {
    if (!out) return SHTC_EINVAL;
    *out = nullptr;
    if (bytes == 0) return SHTC_OK;
    if (cudaHostAlloc(out, bytes, cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        *out = nullptr;
        return SHTC_ENOMEM;
    }
    return SHTC_OK;
}

void shtc_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

shtc_status shtc_plan_executed(shtc_ctx* ctx, uint64_t* alm2map, uint64_t* map2alm) {
    if (!ctx) return SHTC_EINVAL;
    return guarded(ctx, [&] {
        ensure_leg_plan(ctx);
        if (alm2map) *alm2map = ctx->leg.executed_a2m;
        if (map2alm) *map2alm = ctx->leg.executed;
    });
}

shtc_status shtc_alm2map_dev(shtc_ctx* ctx, const double* alm_dev, double* map_dev, shtc_timing* t) {
    if (!ctx || !alm_dev || !map_dev) return SHTC_EINVAL;
    return guarded(ctx, [&] { do_alm2map_dev(ctx, alm_dev, map_dev, t); });
}

shtc_status shtc_map2alm_dev(shtc_ctx* ctx, const double* map_dev, double* alm_dev, shtc_timing* t) {
    if (!ctx || !map_dev || !alm_dev) return SHTC_EINVAL;
    return guarded(ctx, [&] { do_map2alm_dev(ctx, map_dev, alm_dev, t); });
}

// Host-buffer entry points, pipelined over latitude bands (contiguous tile ranges of ~equal
// pixel counts, see tile_bands).  Streams: h2d / d2h copies, two Legendre streams that
// consecutive launches alternate between (one launch's tail overlaps the next launch), and a
// high-priority ring-stage stream whose blocks take the SMs the Legendre launches free.
//   alm2map: H2D of a_lm by order chunk || Legendre of band 0 by order chunk, then the other
//            bands' Legendre launches; ring synthesis of band k after band k's launches ->
//            D2H of the band's pixels
//   map2alm: H2D of band k's pixels -> ring analysis of band k -> band k's Legendre launches
//            (the last band split by order chunk); after launch j (and j-1, the only launch
//            that can still run beside it) the orders whose last item was in launch j are
//            final -> D2H of their a_lm
// Same kernels and arithmetic as the device-resident path (results are bit-identical).
namespace {
void ensure_pipe(shtc_ctx* c) {
    if (c->h2d) return;
    int least = 0, greatest = 0;
    CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    CK(cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking));
    for (auto& st : c->lst) CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithPriority(&c->fst, cudaStreamNonBlocking, greatest));
    for (auto& e : c->pev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : c->tev) CK(cudaEventCreate(&e));
}

// events of one pipelined call, handed out in order
struct PipeEvents {
    shtc_ctx* c;
    int np = 0, nt = 0;
    cudaEvent_t order(cudaStream_t st) {
        if (np >= kPipeEvents) fail(SHTC_ECUDA, "pipeline event pool exhausted");
        cudaEvent_t e = c->pev[np++];
        CK(cudaEventRecord(e, st));
        return e;
    }
    // (start, end) timing pair around enqueue(), recorded on st; returns the pair's index
    int timed(cudaStream_t st, const std::function<void()>& enqueue) {
        if (nt + 2 > kPipeEvents) fail(SHTC_ECUDA, "pipeline event pool exhausted");
        const int i = nt;
        CK(cudaEventRecord(c->tev[nt++], st));
        enqueue();
        CK(cudaEventRecord(c->tev[nt++], st));
        return i;
    }
    float span(int i) const { return elapsed(c->tev[i], c->tev[i + 1]); }
    // SHTC_PIPE_TRACE=1: every timed segment as (start, end) ms after the call's start event
    void trace(const char* what, const std::vector<std::pair<const char*, int>>& segs) const {
        static const bool on = std::getenv("SHTC_PIPE_TRACE") != nullptr;
        if (!on) return;
        std::fprintf(stderr, "[pipe %s]", what);
        for (const auto& sg : segs)
            std::fprintf(stderr, " %s %.3f-%.3f", sg.first, elapsed(c->ev[3], c->tev[sg.second]),
                         elapsed(c->ev[3], c->tev[sg.second + 1]));
        std::fprintf(stderr, " end %.3f\n", elapsed(c->ev[3], c->ev[6]));
    }
};

// band-ordered items [begin, end) of one pipelined launch
LegPlanView items_view(const LegPlan& P, int begin, int end, bool a2m) {
    LegPlanView v = P.band_view;
    if (a2m) {
        v.a2m_items = P.band_view.a2m_items + begin;
        v.n_a2m_items = end - begin;
    } else {
        v.m2a_items = P.band_view.m2a_items + begin;
        v.n_m2a_items = end - begin;
    }
    return v;
}

// complex-element range of order indices [mi0, mi1) in the m-major a_lm triangle (full band)
std::pair<size_t, size_t> alm_span(const shtc_ctx* c, int mi0, int mi1) {
    auto off = [&](int mi) {
        return mi >= (int)c->ms.size() ? alm_count(c->lmax, c->mmax)
                                       : (size_t)alm_offset(c->ms[mi], c->lmax);
    };
    return {off(mi0), off(mi1)};
}

// fork the pipeline streams off the caller's stream
void pipe_fork(shtc_ctx* c) {
    CK(cudaEventRecord(c->ev[3], c->stream));
    for (cudaStream_t st : {c->h2d, c->d2h, c->lst[0], c->lst[1], c->fst})
        CK(cudaStreamWaitEvent(st, c->ev[3], 0));
}

// join: every stream's work precedes the last D2H; the caller's stream continues after it
void pipe_join(shtc_ctx* c) {
    for (cudaStream_t st : {c->h2d, c->lst[0], c->lst[1], c->fst}) {
        CK(cudaEventRecord(c->ev[5], st));
        CK(cudaStreamWaitEvent(c->d2h, c->ev[5], 0));
    }
    CK(cudaEventRecord(c->ev[6], c->d2h));
    CK(cudaStreamWaitEvent(c->stream, c->ev[6], 0));
    CK(cudaEventSynchronize(c->ev[6]));
}
}  // namespace

shtc_status shtc_alm2map(shtc_ctx* ctx, const double* alm, double* map, shtc_timing* t) {
    if (!ctx || !alm || !map) return SHTC_EINVAL;
    return guarded(ctx, [&] {
        require_full_band(ctx);
        ensure_leg_plan(ctx);
        ensure_fft_id(ctx);
        ensure_id_layout(ctx);
        ensure_pipe(ctx);
        const size_t na = alm_count(ctx->lmax, ctx->mmax) * sizeof(double2);
        const size_t nb = (size_t)ctx->npix * sizeof(double);
        ctx->alm_buf.ensure(na);
        ctx->map_buf.ensure(nb);
        ctx->delta.ensure((size_t)ctx->n_rings * (ctx->mmax + 1) * sizeof(double2));
        LegPlan& P = ctx->leg;
        FftPlan& F = ctx->fft_id;
        double2* ab = ctx->alm_buf.as<double2>();
        double* mb = ctx->map_buf.as<double>();
        double2* dl = ctx->delta.as<double2>();
        const int64_t* ro = ctx->id_row_off.as<int64_t>();
        const int n_m = (int)ctx->ms.size();
        int* queues = P.counters.as<int>() + 1 + n_m;  // one word per launch
        // pageable host buffers (the C++ drop-in's std::vectors) go through page-locked
        // staging: a_lm chunks are copied in on all host cores just before their H2D, band
        // pixels are copied out as each band's D2H completes, both overlapping the GPU work
        const bool in_pinned = host_pinned(alm), out_pinned = host_pinned(map);
        const double2* alm_src = reinterpret_cast<const double2*>(alm);
        if (!in_pinned) {
            ctx->stage_alm.ensure(na);
            alm_src = ctx->stage_alm.as<double2>();
        }
        double* map_dst = map;
        if (!out_pinned) {
            ctx->stage_map.ensure(nb);
            map_dst = ctx->stage_map.as<double>();
        }
        PipeEvents E{ctx};
        if (!P.a2m_launch.empty())
            CK(cudaMemsetAsync(queues, 0, P.a2m_launch.size() * sizeof(int), ctx->stream));
        pipe_fork(ctx);
        // SHTC_PIPE_MODE (experiments): 2 (default) = everything on one stream, band by band (the
        // ring synthesis needs whole SMs, which a running persistent Legendre launch never
        // frees); 0 = Legendre launches run ahead on two streams (measured slower)
        static const int mode = std::getenv("SHTC_PIPE_MODE") ? std::atoi(std::getenv("SHTC_PIPE_MODE")) : 2;
        std::vector<int> t_leg, t_fft;
        std::vector<std::pair<const char*, int>> segs;
        int t_d2h_first = -1;
        std::vector<std::vector<size_t>> band_launches(kPipeBands);
        for (size_t q = 0; q < P.a2m_launch.size(); ++q) band_launches[P.a2m_launch[q].tc].push_back(q);
        std::vector<cudaEvent_t> band_done(kPipeBands);
        auto leg_launch = [&](size_t j, cudaEvent_t ready) {
            const auto& L = P.a2m_launch[j];
            cudaStream_t st = mode == 2 ? ctx->fst : ctx->lst[j & 1];
            CK(cudaStreamWaitEvent(st, ready, 0));
            t_leg.push_back(E.timed(st, [&] {
                launch_leg_alm2map(items_view(P, L.begin, L.end, true), ab, dl, ro, queues + j, st,
                                   LEG_PHASE_MAIN | LEG_PHASE_NO_RESET);
                CK(cudaGetLastError());
            }));
            if (st != ctx->fst) CK(cudaStreamWaitEvent(ctx->fst, E.order(st), 0));
        };
        // dead tiles' Delta rows (disjoint from every launch's rows) ahead of the ring stage
        launch_leg_alm2map(P.view, ab, dl, ro, P.counters.as<int>(), ctx->fst, LEG_PHASE_ZERO);
        CK(cudaGetLastError());
        // a_lm by order chunk; the head bands' launches of chunk k follow its copy
        std::vector<cudaEvent_t> h_chunk(kOrderChunks);
        int th = -1, th_last = -1;
        for (int k = 0; k < kOrderChunks; ++k) {
            const auto span = alm_span(ctx, P.chunk_mi[k], P.chunk_mi[k + 1]);
            const size_t b = span.first, e = span.second;  // (a lambda below captures them)
            if (!in_pinned && e > b)
                par_memcpy(ctx->stage_alm.as<double2>() + b, reinterpret_cast<const double2*>(alm) + b,
                           (e - b) * sizeof(double2));
            const int ti = E.timed(ctx->h2d, [&] {
                if (e > b)
                    CK(cudaMemcpyAsync(ab + b, alm_src + b, (e - b) * sizeof(double2), cudaMemcpyHostToDevice,
                                       ctx->h2d));
            });
            if (th < 0) th = ti;
            th_last = ti;
            h_chunk[k] = E.order(ctx->h2d);
            for (size_t j : band_launches[0])
                if (P.a2m_launch[j].mc == k) leg_launch(j, h_chunk[k]);
        }
        // band order: the head bands at the equator first (their launches ran by order chunk
        // above), then from the pole back toward the equator, so the last band before the
        // final copy has the cheap belt-ring synthesis (SHTC_A2M_ORDER=0: ascending)
        static const bool polar_early = !std::getenv("SHTC_A2M_ORDER") || std::atoi(std::getenv("SHTC_A2M_ORDER"));
        const int nh = a2m_head_bands();
        std::vector<int> band_order(kPipeBands);
        for (int k = 0; k < kPipeBands; ++k) band_order[k] = (!polar_early || k < nh) ? k : kPipeBands - 1 - (k - nh);
        std::vector<int> copied;  // bands whose pixels go down, in order
        for (int tc : band_order) {
            if (tc != 0)
                for (size_t j : band_launches[tc]) leg_launch(j, h_chunk[kOrderChunks - 1]);
            if (F.band_pix[tc].empty() && band_launches[tc].empty()) continue;
            t_fft.push_back(E.timed(ctx->fst, [&] { run_ring_synth(ctx, F, dl, mb, nullptr, nullptr, tc, ctx->fst); }));
            CK(cudaStreamWaitEvent(ctx->d2h, E.order(ctx->fst), 0));
            const int ti = E.timed(ctx->d2h, [&] {
                for (const auto& iv : F.band_pix[tc])
                    CK(cudaMemcpyAsync(map_dst + iv.first, mb + iv.first, (iv.second - iv.first) * sizeof(double),
                                       cudaMemcpyDeviceToHost, ctx->d2h));
            });
            band_done[tc] = E.order(ctx->d2h);
            copied.push_back(tc);
            if (t_d2h_first < 0) t_d2h_first = ti;
            segs.push_back({"D", ti});
        }
        if (!out_pinned)
            for (int tc : copied) {
                CK(cudaEventSynchronize(band_done[tc]));
                for (const auto& iv : F.band_pix[tc])
                    par_memcpy(map + iv.first, map_dst + iv.first, (iv.second - iv.first) * sizeof(double));
            }
        pipe_join(ctx);
        {
            for (int i : t_leg) segs.push_back({"L", i});
            for (int i : t_fft) segs.push_back({"F", i});
            E.trace("alm2map", segs);
        }
        if (t) {
            float leg = 0.f, fft = 0.f;
            for (int i : t_leg) leg += E.span(i);
            for (int i : t_fft) fft += E.span(i);
            const float d2h = t_d2h_first < 0 ? 0.f : elapsed(ctx->tev[t_d2h_first], ctx->ev[6]);
            const float h2d = th < 0 ? 0.f : elapsed(ctx->tev[th], ctx->tev[th_last + 1]);
            fill_timing(t, leg, fft, h2d, d2h, elapsed(ctx->ev[3], ctx->ev[6]), P, true);
        }
    });
}

shtc_status shtc_map2alm(shtc_ctx* ctx, const double* map, double* alm, shtc_timing* t) {
    if (!ctx || !alm || !map) return SHTC_EINVAL;
    return guarded(ctx, [&] {
        require_full_band(ctx);
        ensure_leg_plan(ctx);
        ensure_fft_id(ctx);
        ensure_id_layout(ctx);
        ensure_pipe(ctx);
        const size_t na = alm_count(ctx->lmax, ctx->mmax) * sizeof(double2);
        const size_t nb = (size_t)ctx->npix * sizeof(double);
        ctx->alm_buf.ensure(na);
        ctx->map_buf.ensure(nb);
        ctx->delta.ensure((size_t)ctx->n_rings * (ctx->mmax + 1) * sizeof(double2));
        LegPlan& P = ctx->leg;
        FftPlan& F = ctx->fft_id;
        double* mb = ctx->map_buf.as<double>();
        double2* dl = ctx->delta.as<double2>();
        const int64_t* ro = ctx->id_row_off.as<int64_t>();
        const int n_m = (int)ctx->ms.size();
        double2* ab = ctx->alm_buf.as<double2>();
        int* queues = P.counters.as<int>() + 1 + n_m + P.a2m_launch.size();  // one word per launch
        // pageable host buffers go through page-locked staging (see shtc_alm2map): each band's
        // pixels are copied in on all host cores just before its H2D, each launch's final
        // orders are copied out as their D2H completes
        const bool in_pinned = host_pinned(map), out_pinned = host_pinned(alm);
        const double* map_src = map;
        if (!in_pinned) {
            ctx->stage_map.ensure(nb);
            map_src = ctx->stage_map.as<double>();
        }
        double2* alm_dst = reinterpret_cast<double2*>(alm);
        if (!out_pinned) {
            ctx->stage_alm.ensure(na);
            alm_dst = ctx->stage_alm.as<double2>();
        }
        PipeEvents E{ctx};
        if (!P.m2a_launch.empty())
            CK(cudaMemsetAsync(queues, 0, P.m2a_launch.size() * sizeof(int), ctx->stream));
        pipe_fork(ctx);
        int th = -1, th_last = -1;
        auto band_h2d = [&](int tc) {
            if (!in_pinned)
                for (const auto& iv : F.band_pix[tc])
                    par_memcpy(ctx->stage_map.as<double>() + iv.first, map + iv.first,
                               (iv.second - iv.first) * sizeof(double));
            const int ti = E.timed(ctx->h2d, [&] {
                for (const auto& iv : F.band_pix[tc])
                    CK(cudaMemcpyAsync(mb + iv.first, map_src + iv.first, (iv.second - iv.first) * sizeof(double),
                                       cudaMemcpyHostToDevice, ctx->h2d));
            });
            if (th < 0) th = ti;
            th_last = ti;
            return E.order(ctx->h2d);
        };
        // SHTC_M2A_MODE (experiments): 0 (default) = Legendre launches alternate over two
        // streams (one launch's tail overlaps the next) beside the high-priority ring analysis;
        // 2 = analysis and launches band by band on one stream (measured slower: 14.0 against
        // 13.4 ms at C4)
        static const int mode = std::getenv("SHTC_M2A_MODE") ? std::atoi(std::getenv("SHTC_M2A_MODE")) : 0;
        const bool serial = mode == 2;
        // orders without alive tiles are zero: ahead of launch 0 (their copy follows it)
        launch_leg_map2alm(P.view, dl, ro, ab, 0, P.counters.as<int>(), P.m2a_scratch.as<double2>(),
                           serial ? ctx->fst : ctx->lst[0], LEG_PHASE_ZERO);
        CK(cudaGetLastError());
        std::vector<int> t_fft, t_leg;
        std::vector<std::pair<const char*, int>> segs;
        int t_d2h_first = -1;
        cudaEvent_t prev = nullptr;
        std::vector<std::pair<int, cudaEvent_t>> d2h_done;  // (launch, its copies done)
        auto copy_final = [&](int j) {
            const int ti = E.timed(ctx->d2h, [&] {
                for (const auto& run : P.m2a_done[j]) {
                    auto [b, e] = alm_span(ctx, run.first, run.second);
                    if (e > b)
                        CK(cudaMemcpyAsync(alm_dst + b, ab + b, (e - b) * sizeof(double2), cudaMemcpyDeviceToHost,
                                           ctx->d2h));
                }
            });
            d2h_done.push_back({j, E.order(ctx->d2h)});
            if (t_d2h_first < 0) t_d2h_first = ti;
            segs.push_back({"D", ti});
        };
        if (P.m2a_launch.empty()) {
            CK(cudaStreamWaitEvent(ctx->d2h, E.order(serial ? ctx->fst : ctx->lst[0]), 0));
            copy_final(0);
        }
        size_t j = 0;
        for (int tc = 0; tc < kPipeBands; ++tc) {
            CK(cudaStreamWaitEvent(ctx->fst, band_h2d(tc), 0));
            t_fft.push_back(E.timed(ctx->fst, [&] { run_ring_anal(ctx, F, mb, dl, nullptr, nullptr, tc, nullptr, ctx->fst); }));
            cudaEvent_t anal_done = serial ? nullptr : E.order(ctx->fst);
            for (; j < P.m2a_launch.size() && P.m2a_launch[j].tc == tc; ++j) {
                const auto& L = P.m2a_launch[j];
                cudaStream_t st = serial ? ctx->fst : ctx->lst[j & 1];
                if (anal_done) CK(cudaStreamWaitEvent(st, anal_done, 0));
                t_leg.push_back(E.timed(st, [&] {
                    launch_leg_map2alm(items_view(P, L.begin, L.end, false), dl, ro, ab, 0, queues + j,
                                       P.m2a_scratch.as<double2>(), st, LEG_PHASE_MAIN | LEG_PHASE_NO_RESET);
                    CK(cudaGetLastError());
                }));
                // the launch's final orders: their items ran in this launch and earlier ones
                // (launch j - 1 may still run beside it on the other stream)
                if (prev && !serial) CK(cudaStreamWaitEvent(st, prev, 0));
                prev = E.order(st);
                launch_leg_m2a_finalize(P.band_view, P.m2a_final_list.as<int>() + P.m2a_final_off[j],
                                        P.m2a_final_off[j + 1] - P.m2a_final_off[j], P.m2a_scratch.as<double2>(),
                                        ab, 0, st);
                CK(cudaGetLastError());
                CK(cudaStreamWaitEvent(ctx->d2h, E.order(st), 0));
                copy_final((int)j);
            }
        }
        if (!out_pinned)
            for (const auto& [jj, ev] : d2h_done) {
                CK(cudaEventSynchronize(ev));
                for (const auto& run : P.m2a_done[jj]) {
                    auto [b, e] = alm_span(ctx, run.first, run.second);
                    if (e > b)
                        par_memcpy(reinterpret_cast<double2*>(alm) + b, alm_dst + b, (e - b) * sizeof(double2));
                }
            }
        pipe_join(ctx);
        {
            for (int i : t_leg) segs.push_back({"L", i});
            for (int i : t_fft) segs.push_back({"F", i});
            E.trace("map2alm", segs);
        }
        if (t) {
            float leg = 0.f, fft = 0.f;
            for (int i : t_leg) leg += E.span(i);
            for (int i : t_fft) fft += E.span(i);
            const float d2h = t_d2h_first < 0 ? 0.f : elapsed(ctx->tev[t_d2h_first], ctx->ev[6]);
            const float h2d = th < 0 ? 0.f : elapsed(ctx->tev[th], ctx->tev[th_last + 1]);
            fill_timing(t, leg, fft, h2d, d2h, elapsed(ctx->ev[3], ctx->ev[6]), P, false);
        }
    });
}

// ---- stage API -------------------------------------------------------------------------
shtc_status shtc_set_exchange_layout(shtc_ctx* ctx, const int64_t* row_off, int n_ring_list,
                                     const int32_t* ring_list, const int64_t* m_base,
                                     const int64_t* m_stride) {
    if (!ctx) return SHTC_EINVAL;
    return guarded(ctx, [&] {
        if (!ctx->grid_set || !ctx->band_set) fail(SHTC_EINVAL, "set grid and band first");
        ctx->peers_set = false;  // the peer targets are rebuilt on top of the new layout
        ctx->syn_layout = false;
        if (!row_off) {
            ctx->custom_layout = false;
            return;
        }
        if (n_ring_list < 0 || (n_ring_list > 0 && (!ring_list || !m_base || !m_stride)))
            fail(SHTC_EINVAL, "exchange layout: malformed");
        ctx->row_off.assign(row_off, row_off + ctx->n_rings);
        ctx->ring_list.assign(ring_list, ring_list + n_ring_list);
        for (int i = 0; i < n_ring_list; ++i) {
            if (ring_list[i] < 0 || ring_list[i] >= ctx->n_rings)
                fail(SHTC_EINVAL, "exchange: invalid ring layout");
            if (i > 0 && ring_list[i] <= ring_list[i - 1])
                fail(SHTC_EINVAL, "exchange: ring list must be ascending");
        }
        ctx->m_base.assign(m_base, m_base + ctx->mmax + 1);
        ctx->m_stride.assign(m_stride, m_stride + ctx->mmax + 1);
        ctx->row_off_d.upload(ctx->row_off, ctx->stream);
        ctx->m_base_d.upload(ctx->m_base, ctx->stream);
        ctx->m_stride_d.upload(ctx->m_stride, ctx->stream);
        std::vector<int> order(ctx->mmax + 1);
        std::iota(order.begin(), order.end(), 0);
        std::stable_sort(order.begin(), order.end(),
                         [&](int x, int y) { return ctx->m_base[x] < ctx->m_base[y]; });
        // (SHTC_UNFOLD_ASCENDING=1: ascending m, the comparison order for the coalescing
        // measurement in tools/exchange_coalesce.py)
        static const bool ascending = std::getenv("SHTC_UNFOLD_ASCENDING") && std::atoi(std::getenv("SHTC_UNFOLD_ASCENDING"));
        if (ascending) std::iota(order.begin(), order.end(), 0);
        ctx->m_order_d.upload(order, ctx->stream);
        build_fft_plan(ctx, ctx->fft_custom, ctx->ring_list);
        ctx->custom_layout = true;
    });
}

shtc_status shtc_set_exchange_layout_synthesis(shtc_ctx* ctx, const int64_t* row_off, const int64_t* row_stride,
                                               const int64_t* m_base, const int64_t* m_stride) {
    if (!ctx) return SHTC_EINVAL;
    return guarded(ctx, [&] {
        ctx->peers_set = false;  // row_ptr targets are read with this layout's strides
        if (!row_off) {
            ctx->syn_layout = false;
            return;
        }
        if (!ctx->custom_layout) fail(SHTC_EINVAL, "exchange layout (synthesis): set the exchange layout first");
        if (!row_stride || !m_base || !m_stride) fail(SHTC_EINVAL, "exchange layout (synthesis): malformed");
        ctx->syn_row_off_d.upload(std::vector<int64_t>(row_off, row_off + ctx->n_rings), ctx->stream);
        ctx->syn_row_stride_d.upload(std::vector<int64_t>(row_stride, row_stride + ctx->n_rings), ctx->stream);
        ctx->syn_m_base_d.upload(std::vector<int64_t>(m_base, m_base + ctx->mmax + 1), ctx->stream);
        ctx->syn_m_stride_d.upload(std::vector<int64_t>(m_stride, m_stride + ctx->mmax + 1), ctx->stream);
        CK(cudaStreamSynchronize(ctx->stream));
        ctx->syn_layout = true;
    });
}

namespace {
const int64_t* stage_row_off(shtc_ctx* c) {
    if (c->custom_layout) return c->row_off_d.as<int64_t>();
    ensure_id_layout(c);
    return c->id_row_off.as<int64_t>();
}
}  // namespace

shtc_status shtc_legendre_alm2map_dev(shtc_ctx* ctx, const double* alm_dev, double* delta_dev,
                                      shtc_timing* t) {
    if (!ctx || !alm_dev || !delta_dev) return SHTC_EINVAL;
    return guarded(ctx, [&] {
        ensure_leg_plan(ctx);
        const int64_t* ro = ctx->syn_layout ? ctx->syn_row_off_d.as<int64_t>() : stage_row_off(ctx);
        LegPlanView v = ctx->leg.view;
        if (ctx->syn_layout) v.row_stride = ctx->syn_row_stride_d.as<int64_t>();
        CK(cudaEventRecord(ctx->ev[0], ctx->stream));
        launch_leg_alm2map(v, reinterpret_cast<const double2*>(alm_dev),
                           reinterpret_cast<double2*>(delta_dev), ro, ctx->leg.counters.as<int>(),
                           ctx->stream);
        CK(cudaGetLastError());
        CK(cudaEventRecord(ctx->ev[1], ctx->stream));
        if (t) {
            CK(cudaEventSynchronize(ctx->ev[1]));
            const double leg = elapsed(ctx->ev[0], ctx->ev[1]);
            fill_timing(t, leg, 0, 0, 0, leg, ctx->leg, true);
        }
    });
}

shtc_status shtc_legendre_map2alm_dev(shtc_ctx* ctx, const double* delta_dev, double* alm_dev,
                                      shtc_timing* t) {
    if (!ctx || !alm_dev || !delta_dev) return SHTC_EINVAL;
    return guarded(ctx, [&] {
        ensure_leg_plan(ctx);
        const int64_t* ro = stage_row_off(ctx);
        CK(cudaEventRecord(ctx->ev[0], ctx->stream));
        launch_leg_map2alm(ctx->leg.view, reinterpret_cast<const double2*>(delta_dev), ro,
                           reinterpret_cast<double2*>(alm_dev), 0, ctx->leg.counters.as<int>(),
                           ctx->leg.m2a_scratch.as<double2>(), ctx->stream);
        CK(cudaGetLastError());
        CK(cudaEventRecord(ctx->ev[1], ctx->stream));
        if (t) {
            CK(cudaEventSynchronize(ctx->ev[1]));
            const double leg = elapsed(ctx->ev[0], ctx->ev[1]);
            fill_timing(t, leg, 0, 0, 0, leg, ctx->leg, false);
        }
    });
}

shtc_status shtc_ring_synthesis_dev(shtc_ctx* ctx, const double* delta_dev, double* map_dev,
                                    shtc_timing* t) {
    if (!ctx || !delta_dev || !map_dev) return SHTC_EINVAL;
    return guarded(ctx, [&] {
        FftPlan* F;
        const int64_t *mb, *mst;
        if (ctx->custom_layout) {
            F = &ctx->fft_custom;
            mb = (ctx->syn_layout ? ctx->syn_m_base_d : ctx->m_base_d).as<int64_t>();
            mst = (ctx->syn_layout ? ctx->syn_m_stride_d : ctx->m_stride_d).as<int64_t>();
        } else {
            require_full_band(ctx);
            ensure_fft_id(ctx);
            ensure_id_layout(ctx);
            F = &ctx->fft_id;
            mb = nullptr;
            mst = nullptr;
        }
        CK(cudaEventRecord(ctx->ev[0], ctx->stream));
        run_ring_synth(ctx, *F, reinterpret_cast<const double2*>(delta_dev), map_dev, mb, mst);
        CK(cudaEventRecord(ctx->ev[1], ctx->stream));
        if (t) {
            CK(cudaEventSynchronize(ctx->ev[1]));
            *t = shtc_timing{};
            t->fft_ms = t->total_ms = elapsed(ctx->ev[0], ctx->ev[1]);
        }
    });
}

shtc_status shtc_ring_analysis_dev(shtc_ctx* ctx, const double* map_dev, double* delta_dev,
                                   shtc_timing* t) {
    if (!ctx || !delta_dev || !map_dev) return SHTC_EINVAL;
    return guarded(ctx, [&] {
        FftPlan* F;
        const int64_t *mb, *mst;
        if (ctx->custom_layout) {
            F = &ctx->fft_custom;
            mb = ctx->m_base_d.as<int64_t>();
            mst = ctx->m_stride_d.as<int64_t>();
        } else {
            require_full_band(ctx);
            ensure_fft_id(ctx);
            ensure_id_layout(ctx);
            F = &ctx->fft_id;
            mb = nullptr;
            mst = nullptr;
        }
        CK(cudaEventRecord(ctx->ev[0], ctx->stream));
        run_ring_anal(ctx, *F, map_dev, reinterpret_cast<double2*>(delta_dev), mb, mst, -1, nullptr, nullptr,
                      ctx->custom_layout ? ctx->m_order_d.as<int>() : nullptr);
        CK(cudaEventRecord(ctx->ev[1], ctx->stream));
        if (t) {
            CK(cudaEventSynchronize(ctx->ev[1]));
            *t = shtc_timing{};
            t->fft_ms = t->total_ms = elapsed(ctx->ev[0], ctx->ev[1]);
        }
    });
}

// ---- fused exchange over peer memory ----------------------------------------------------
// exchange_m_to_rings / exchange_rings_to_m (distribution.cpp:233-298) as direct stores from
// the producing kernels into the consumers' buffers, then one device-side barrier.
shtc_status shtc_dev_alloc(int device, uint64_t bytes, void** ptr) {
    if (!ptr || bytes == 0) return SHTC_EINVAL;
    return guarded(nullptr, [&] {
        CK(cudaSetDevice(device));
        void* p = nullptr;
        if (cudaMalloc(&p, bytes) != cudaSuccess) {
            cudaGetLastError();
            fail(SHTC_ENOMEM, "shtc_dev_alloc: cudaMalloc failed");
        }
        CK(cudaMemset(p, 0, bytes));
        *ptr = p;
    });
}

shtc_status shtc_dev_free(void* ptr) {
    return guarded(nullptr, [&] {
        if (ptr) CK(cudaFree(ptr));
    });
}

shtc_status shtc_ipc_handle(const void* ptr, unsigned char* handle64) {
    if (!ptr || !handle64) return SHTC_EINVAL;
    return guarded(nullptr, [&] {
        cudaIpcMemHandle_t h;
        CK(cudaIpcGetMemHandle(&h, const_cast<void*>(ptr)));
        static_assert(sizeof(h) == 64, "CUDA IPC handle size");
        std::memcpy(handle64, &h, 64);
    });
}

shtc_status shtc_ipc_open(int device, const unsigned char* handle64, void** ptr) {
    if (!handle64 || !ptr) return SHTC_EINVAL;
    return guarded(nullptr, [&] {
        CK(cudaSetDevice(device));
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle64, 64);
        CK(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
    });
}

shtc_status shtc_ipc_close(void* ptr) {
    return guarded(nullptr, [&] {
        if (ptr) CK(cudaIpcCloseMemHandle(ptr));
    });
}

shtc_status shtc_set_exchange_peers(shtc_ctx* ctx, const uint64_t* row_ptr, const uint64_t* col_ptr) {
    if (!ctx) return SHTC_EINVAL;
    return guarded(ctx, [&] {
        if (!row_ptr || !col_ptr) {
            ctx->peers_set = false;
            return;
        }
        if (!ctx->custom_layout) fail(SHTC_EINVAL, "exchange peers: set the exchange layout first");
        std::vector<uint64_t> rp(row_ptr, row_ptr + ctx->n_rings), cp(col_ptr, col_ptr + ctx->mmax + 1);
        ctx->peer_row_ptr.upload(rp, ctx->stream);
        ctx->peer_col_ptr.upload(cp, ctx->stream);
        CK(cudaStreamSynchronize(ctx->stream));
        ctx->peers_set = true;
    });
}

shtc_status shtc_legendre_alm2map_peer(shtc_ctx* ctx, const double* alm_dev, shtc_timing* t) {
    if (!ctx || !alm_dev) return SHTC_EINVAL;
    return guarded(ctx, [&] {
        if (!ctx->peers_set || !ctx->custom_layout || !ctx->fft_custom.built)
            fail(SHTC_EINVAL, "exchange peers not set");
        ensure_leg_plan(ctx);
        LegPlanView v = ctx->leg.view;
        v.row_ptr = ctx->peer_row_ptr.as<double2*>();
        if (ctx->syn_layout) v.row_stride = ctx->syn_row_stride_d.as<int64_t>();
        CK(cudaEventRecord(ctx->ev[0], ctx->stream));
        launch_leg_alm2map(v, reinterpret_cast<const double2*>(alm_dev), nullptr,
                           (ctx->syn_layout ? ctx->syn_row_off_d : ctx->row_off_d).as<int64_t>(),
                           ctx->leg.counters.as<int>(), ctx->stream);
        CK(cudaGetLastError());
        CK(cudaEventRecord(ctx->ev[1], ctx->stream));
        if (t) {
            CK(cudaEventSynchronize(ctx->ev[1]));
            const double leg = elapsed(ctx->ev[0], ctx->ev[1]);
            fill_timing(t, leg, 0, 0, 0, leg, ctx->leg, true);
        }
    });
}

shtc_status shtc_ring_analysis_peer(shtc_ctx* ctx, const double* map_dev, shtc_timing* t) {
    if (!ctx || !map_dev) return SHTC_EINVAL;
    return guarded(ctx, [&] {
        if (!ctx->peers_set || !ctx->custom_layout || !ctx->fft_custom.built)
            fail(SHTC_EINVAL, "exchange peers not set");
        CK(cudaEventRecord(ctx->ev[0], ctx->stream));
        run_ring_anal(ctx, ctx->fft_custom, map_dev, nullptr, ctx->m_base_d.as<int64_t>(),
                      ctx->m_stride_d.as<int64_t>(), -1, ctx->peer_col_ptr.as<double2*>(), nullptr,
                      ctx->m_order_d.as<int>());
        CK(cudaEventRecord(ctx->ev[1], ctx->stream));
        if (t) {
            CK(cudaEventSynchronize(ctx->ev[1]));
            *t = shtc_timing{};
            t->fft_ms = t->total_ms = elapsed(ctx->ev[0], ctx->ev[1]);
        }
    });
}

shtc_status shtc_peer_barrier(shtc_ctx* ctx, int rank, int n_workers, const uint64_t* flags,
                              uint32_t epoch) {
    if (!ctx || !flags || n_workers < 1 || n_workers > PEER_MAX || rank < 0 || rank >= n_workers)
        return SHTC_EINVAL;
    return guarded(ctx, [&] {
        PeerFlags f{};
        for (int w = 0; w < n_workers; ++w) {
            if (!flags[w]) fail(SHTC_EINVAL, "peer barrier: null flag array");
            f.f[w] = reinterpret_cast<unsigned int*>(flags[w]);
        }
        launch_peer_barrier(f, rank, n_workers, epoch, ctx->stream);
        CK(cudaGetLastError());
    });
}

shtc_status shtc_copy_orders(shtc_ctx* ctx, const double* src, double* dst, int to_device) {
    if (!ctx || !src || !dst) return SHTC_EINVAL;
    return guarded(ctx, [&] {
        if (!ctx->band_set) fail(SHTC_EINVAL, "no band set");
        const cudaMemcpyKind kind = to_device ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
        const double2* s2 = reinterpret_cast<const double2*>(src);
        double2* d2 = reinterpret_cast<double2*>(dst);
        for (size_t i = 0; i < ctx->ms.size();) {
            // runs of consecutive orders are contiguous in the triangle: one copy per run
            size_t e = i + 1;
            while (e < ctx->ms.size() && ctx->ms[e] == ctx->ms[e - 1] + 1) ++e;
            const size_t b0 = (size_t)alm_offset(ctx->ms[i], ctx->lmax);
            const size_t b1 = (size_t)alm_offset(ctx->ms[e - 1], ctx->lmax) + (ctx->lmax - ctx->ms[e - 1] + 1);
            CK(cudaMemcpyAsync(d2 + b0, s2 + b0, (b1 - b0) * sizeof(double2), kind, ctx->stream));
            i = e;
        }
    });
}

// ---- Legendre-stage operators ---------------------------------------------------------
namespace {
void op_plan(shtc_ctx* c, int lmax, int mmax, int n_lat, const double* x, int n_m, const int32_t* ms) {
    std::vector<int> mv(ms, ms + n_m);
    std::vector<double> xv(x, x + n_lat);
    if (c->op_leg.built && c->op_leg.lmax == lmax && c->op_leg.ms == mv && c->op_x == xv &&
        c->op_leg.view.unscaled == (c->ladder ? 0 : 1))
        return;
    std::vector<double> lmu(mmax + 1);
    for (int m = 0; m <= mmax; ++m) lmu[m] = host_log_mu(m);
    std::vector<Stream> st(n_lat);
    for (int r = 0; r < n_lat; ++r) st[r] = {x[r], r, -1};
    build_leg_plan(c, c->op_leg, lmax, mmax, mv, st, lmu);
    c->op_x = xv;
}
}  // namespace

shtc_status shtc_delta_a(shtc_ctx* ctx, const double* alm, int lmax, int mmax, int n_lat,
                         const double* x, int n_m, const int32_t* ms, double* delta, uint64_t* steps) {
    if (!ctx) return SHTC_EINVAL;
    return guarded(ctx, [&] {
        if (lmax < mmax || mmax < 0) fail(SHTC_EINVAL, "AlmSet: need lmax >= mmax >= 0");
        if (n_lat < 0 || n_m < 0) fail(SHTC_EINVAL, "compute_delta_a: negative sizes");
        check_m_set(ms, n_m, mmax, "compute_delta_a");
        check_latitudes(x, n_lat, "compute_delta_a");
        uint64_t nominal = 0;
        for (int i = 0; i < n_m; ++i) nominal += (uint64_t)(lmax - ms[i] + 1) * n_lat;
        if (steps) *steps += nominal;
        if (n_lat == 0 || n_m == 0) return;
        op_plan(ctx, lmax, mmax, n_lat, x, n_m, ms);
        cudaStream_t s = ctx->stream;
        const size_t na = alm_count(lmax, mmax) * sizeof(double2);
        const size_t nd = (size_t)n_lat * n_m * sizeof(double2);
        DevBuf a, d, ro;
        a.ensure(na);
        d.ensure(nd);
        std::vector<int64_t> rov(n_lat);
        for (int r = 0; r < n_lat; ++r) rov[r] = (int64_t)r * n_m;
        ro.upload(rov, s);
        CK(cudaMemcpyAsync(a.p, alm, na, cudaMemcpyHostToDevice, s));
        launch_leg_alm2map(ctx->op_leg.view, a.as<double2>(), d.as<double2>(), ro.as<int64_t>(),
                           ctx->op_leg.counters.as<int>(), s);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(delta, d.p, nd, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    });
}

shtc_status shtc_accumulate_alm(shtc_ctx* ctx, const double* delta, int n_lat, const double* x,
                                int n_m, const int32_t* ms, int lmax, int mmax, double* alm_inout,
                                uint64_t* steps) {
    if (!ctx) return SHTC_EINVAL;
    return guarded(ctx, [&] {
        if (lmax < mmax || mmax < 0) fail(SHTC_EINVAL, "accumulate_alm: need lmax >= mmax >= 0");
        if (n_lat < 0 || n_m < 0) fail(SHTC_EINVAL, "accumulate_alm: negative sizes");
        check_latitudes(x, n_lat, "accumulate_alm");
        check_m_set(ms, n_m, mmax, "accumulate_alm: panel order outside [0, mmax]");
        uint64_t nominal = 0;
        for (int i = 0; i < n_m; ++i) nominal += (uint64_t)(lmax - ms[i] + 1) * n_lat;
        if (steps) *steps += nominal;
        if (n_lat == 0 || n_m == 0) return;
        op_plan(ctx, lmax, mmax, n_lat, x, n_m, ms);
        cudaStream_t s = ctx->stream;
        const size_t na = alm_count(lmax, mmax) * sizeof(double2);
        const size_t nd = (size_t)n_lat * n_m * sizeof(double2);
        DevBuf a, d, ro;
        a.ensure(na);
        d.ensure(nd);
        std::vector<int64_t> rov(n_lat);
        for (int r = 0; r < n_lat; ++r) rov[r] = (int64_t)r * n_m;
        ro.upload(rov, s);
        CK(cudaMemcpyAsync(a.p, alm_inout, na, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(d.p, delta, nd, cudaMemcpyHostToDevice, s));
        launch_leg_map2alm(ctx->op_leg.view, d.as<double2>(), ro.as<int64_t>(), a.as<double2>(), 1,
                           ctx->op_leg.counters.as<int>(), ctx->op_leg.m2a_scratch.as<double2>(), s);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(alm_inout, a.p, na, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    });
}

// ---- device helpers --------------------------------------------------------------------
shtc_status shtc_device_info(int device, char* name, int name_len, int* sm_count, int* cc_major,
                             int* cc_minor) {
    return guarded(nullptr, [&] {
        cudaDeviceProp prop{};
        CK(cudaGetDeviceProperties(&prop, device));
        if (name && name_len > 0) {
            std::strncpy(name, prop.name, name_len - 1);
            name[name_len - 1] = 0;
        }
        if (sm_count) *sm_count = prop.multiProcessorCount;
        if (cc_major) *cc_major = prop.major;
        if (cc_minor) *cc_minor = prop.minor;
    });
}

shtc_status shtc_measure_fp64_peak(int device, double* tflops, double* sm_clock_mhz) {
    return guarded(nullptr, [&] {
        CK(cudaSetDevice(device));
        cudaDeviceProp prop{};
        CK(cudaGetDeviceProperties(&prop, device));
        DevBuf out;
        out.ensure(sizeof(double));
        cudaStream_t s;
        CK(cudaStreamCreate(&s));
        cudaEvent_t a, b;
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
        const int blocks = prop.multiProcessorCount * 4, threads = 256, iters = 4096;
        launch_dfma_peak(out.as<double>(), blocks, threads, 64, s);  // warm-up
        CK(cudaEventRecord(a, s));
        launch_dfma_peak(out.as<double>(), blocks, threads, iters, s);
        CK(cudaEventRecord(b, s));
        CK(cudaEventSynchronize(b));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, a, b));
        const double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
        if (tflops) *tflops = flops / (ms * 1e-3) / 1e12;
        if (sm_clock_mhz) {
            int khz = 0;
            cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, device);
            *sm_clock_mhz = khz / 1000.0;
        }
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        cudaStreamDestroy(s);
    });
}

}  // extern "C"
