// libshtc multi-GPU group: the reference's in-process workers (distributed_synthesis /
// distributed_analysis, /root/reference/proj/src/distribution.cpp:300-490) as one process
// driving W device contexts, worker i on device_ids[i].
//
//   alm2map  per worker: H2D of its orders' a_lm -> Legendre stage over all rings x its orders
//            -> Delta exchange m -> rings -> ring synthesis of its rings -> D2H of its pixels
//   map2alm  per worker: H2D of its rings' pixels -> ring analysis -> Delta exchange rings -> m
//            -> Legendre stage of its orders -> D2H of its a_lm
//
// The exchange (exchange_m_to_rings / exchange_rings_to_m, distribution.cpp:233-298) is either
//   * fused (SHTC_EXCHANGE_PEER, the default): the producing kernel stores every Delta entry
//     straight into the consumer's buffer (NVLink peer memory between devices, plain stores
//     when workers share a device), then each consumer stream waits on every producer's
//     completion event -- no pack / unpack kernels, no collective, no spinning; or
//   * NCCL (SHTC_EXCHANGE_NCCL, the measured baseline): ncclCommInitAll over the devices and
//     one grouped ncclSend / ncclRecv per worker pair on the packed buffers the stage kernels
//     read and write in place.  libnccl is dlopen'ed on first use (libshtc links cudart only).
// Results equal the single-context transforms (worker-count invariance, as the reference's).
// This file is host code only: every transform runs through the context's C ABI (shtc.cu).

#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

#include <nccl.h>  // types only; the library is loaded at run time

#include "../../include/shtc.h"
#include "hostutil.h"

namespace {

thread_local std::string g_group_error;

struct GroupError {
    shtc_status code;
    std::string msg;
};

[[noreturn]] void gfail(shtc_status c, const std::string& m) { throw GroupError{c, m}; }

void gck(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        gfail(e == cudaErrorMemoryAllocation ? SHTC_ENOMEM : SHTC_ECUDA,
              std::string(what) + ": " + cudaGetErrorString(e));
}
#define GCK(x) gck((x), #x)

// ---- NCCL, loaded at run time --------------------------------------------------------------
struct Nccl {
    bool ok = false;
    std::string why;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;

    static Nccl& get() {
        static Nccl n = [] {
            Nccl x;
            const char* env = std::getenv("SHTC_NCCL_LIB");
            void* h = nullptr;
            for (const char* name : {env, "libnccl.so.2", "libnccl.so"}) {
                if (!name) continue;
                h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
                if (h) break;
            }
            if (!h) {
                x.why = std::string("NCCL library not found (libnccl.so.2): ") + (dlerror() ?: "");
                return x;
            }
            auto sym = [&](auto& fp, const char* name) {
                fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
                return fp != nullptr;
            };
            x.ok = sym(x.CommInitAll, "ncclCommInitAll") && sym(x.CommDestroy, "ncclCommDestroy") &&
                   sym(x.GroupStart, "ncclGroupStart") && sym(x.GroupEnd, "ncclGroupEnd") &&
                   sym(x.Send, "ncclSend") && sym(x.Recv, "ncclRecv") &&
                   sym(x.GetErrorString, "ncclGetErrorString");
            if (!x.ok) x.why = "NCCL library lacks the point-to-point API";
            return x;
        }();
        return n;
    }
    void check(ncclResult_t r, const char* what) const {
        if (r != ncclSuccess) gfail(SHTC_ECUDA, std::string(what) + ": " + GetErrorString(r));
    }
};

struct Pinned {
    void* p = nullptr;
    size_t bytes = 0;
    ~Pinned() { release(); }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        bytes = 0;
    }
    void ensure(size_t b) {
        if (p && b <= bytes) return;
        release();
        GCK(cudaHostAlloc(&p, b ? b : 16, cudaHostAllocPortable));
        bytes = b;
    }
};

size_t alm_count(int lmax, int mmax) {
    const size_t l = lmax, m = mmax;
    return (m + 1) * (l + 1) - m * (m + 1) / 2;
}
int64_t alm_offset(int m, int lmax) { return (int64_t)m * (lmax + 1) - (int64_t)m * (m - 1) / 2; }

constexpr int kEv = 6;  // start, after H2D, after stage 1, after exchange, after stage 2, done

struct Worker {
    int dev = 0;
    shtc_ctx* ctx = nullptr;
    cudaStream_t s = nullptr;
    cudaEvent_t ev[kEv] = {};
    std::vector<int> ms, rings;
    std::vector<std::pair<int64_t, int64_t>> pix;  // pixel intervals of the worker's rings
    // packed exchange buffers (complex elements): send = Legendre side (blocks per ring owner),
    // recv = ring side (blocks per order owner); per-peer block offsets and counts
    void* send = nullptr;
    void* recv = nullptr;
    std::vector<int64_t> send_off, send_cnt, recv_off, recv_cnt;
    void* a_dev = nullptr;  // full a_lm triangle (the worker reads / writes its orders only)
    void* m_dev = nullptr;  // full map (the worker reads / writes its rings only)
    ncclComm_t comm = nullptr;
    uint64_t nominal = 0;
};

}  // namespace

struct shtc_group {
    int mode = SHTC_EXCHANGE_PEER;
    std::vector<Worker> w;
    std::string err;
    // grid
    int n_rings = 0;
    std::vector<double> cos_theta, phi0, weight;
    std::vector<int32_t> nphi;
    std::vector<int64_t> pixoff;
    int64_t npix = 0;
    int mirror = 1;
    bool grid_set = false;
    // layout
    int lmax = -1, mmax = -1;
    bool layout_set = false;
    bool ran = false;  // a previous call's completion events exist (write-after-read order)
    double plan_ms = 0.0;
    Pinned stage_alm, stage_map;
};

namespace {

void set_gerr(shtc_group* g, const std::string& m) {
    g_group_error = m;
    if (g) g->err = m;
}

template <class F>
shtc_status gguard(shtc_group* g, F&& f) {
    try {
        f();
        return SHTC_OK;
    } catch (const GroupError& e) {
        set_gerr(g, e.msg);
        return e.code;
    } catch (const std::bad_alloc&) {
        set_gerr(g, "host allocation failed");
        return SHTC_ENOMEM;
    } catch (const std::exception& e) {
        set_gerr(g, e.what());
        return SHTC_ECUDA;
    }
}

// a context call that failed: its message, its status
void cck(shtc_status st, const Worker& w, const char* what) {
    if (st != SHTC_OK) gfail(st, std::string(what) + " (worker on device " + std::to_string(w.dev) + "): " +
                                     shtc_last_error(w.ctx));
}

void free_buffers(Worker& w) {
    cudaSetDevice(w.dev);
    for (void** p : {&w.send, &w.recv, &w.a_dev, &w.m_dev})
        if (*p) {
            cudaFree(*p);
            *p = nullptr;
        }
}

void* dev_alloc(int dev, size_t bytes) {
    GCK(cudaSetDevice(dev));
    void* p = nullptr;
    if (cudaMalloc(&p, bytes ? bytes : 16) != cudaSuccess) {
        cudaGetLastError();
        gfail(SHTC_ENOMEM, "shtc_group: device allocation of " + std::to_string(bytes) + " bytes failed");
    }
    return p;
}

// Packed exchange layout of worker i (the layouts of sht.exchange_layout; distribution.cpp:
// 233-298 moves exactly these blocks): send block for ring owner j = |R_j| rows x |M_i| orders,
// recv block from order owner j = |R_i| rows x |M_j| orders.
void build_exchange(shtc_group* g) {
    const int W = (int)g->w.size();
    std::vector<int64_t> M(W), R(W);
    for (int j = 0; j < W; ++j) {
        M[j] = (int64_t)g->w[j].ms.size();
        R[j] = (int64_t)g->w[j].rings.size();
    }
    for (int i = 0; i < W; ++i) {
        Worker& wi = g->w[i];
        wi.send_off.assign(W, 0);
        wi.send_cnt.assign(W, 0);
        wi.recv_off.assign(W, 0);
        wi.recv_cnt.assign(W, 0);
        int64_t so = 0, ro = 0;
        for (int j = 0; j < W; ++j) {
            wi.send_off[j] = so;
            wi.send_cnt[j] = R[j] * M[i];
            so += R[j] * M[i];
            wi.recv_off[j] = ro;
            wi.recv_cnt[j] = R[i] * M[j];
            ro += R[i] * M[j];
        }
        free_buffers(wi);
        wi.send = dev_alloc(wi.dev, (size_t)so * 16);
        wi.recv = dev_alloc(wi.dev, (size_t)ro * 16);
        wi.a_dev = dev_alloc(wi.dev, alm_count(g->lmax, g->mmax) * 16);
        wi.m_dev = dev_alloc(wi.dev, (size_t)g->npix * 8);
        GCK(cudaMemsetAsync(wi.send, 0, (size_t)so * 16, wi.s));
        GCK(cudaMemsetAsync(wi.recv, 0, (size_t)ro * 16, wi.s));
    }
    for (int i = 0; i < W; ++i) {
        Worker& wi = g->w[i];
        std::vector<int64_t> row_off(g->n_rings, 0), m_base(g->mmax + 1, 0), m_stride(g->mmax + 1, 1);
        for (int j = 0; j < W; ++j)
            for (size_t p = 0; p < g->w[j].rings.size(); ++p)
                row_off[g->w[j].rings[p]] = wi.send_off[j] + (int64_t)p * M[i];
        for (int j = 0; j < W; ++j)
            for (size_t c = 0; c < g->w[j].ms.size(); ++c) {
                m_base[g->w[j].ms[c]] = wi.recv_off[j] + (int64_t)c;
                m_stride[g->w[j].ms[c]] = M[j];
            }
        GCK(cudaSetDevice(wi.dev));
        cck(shtc_set_exchange_layout(wi.ctx, row_off.data(), (int)wi.rings.size(), wi.rings.data(), m_base.data(),
                                     m_stride.data()),
            wi, "exchange layout");
        // synthesis direction: the same blocks order-major ([M_i x R_j]), so the Legendre
        // kernel's stores (one order, consecutive rings per warp) are contiguous runs
        std::vector<int64_t> s_row_off(g->n_rings, 0), s_row_stride(g->n_rings, 1), s_m_base(g->mmax + 1, 0),
            s_m_stride(g->mmax + 1, 1);
        for (int j = 0; j < W; ++j)
            for (size_t p = 0; p < g->w[j].rings.size(); ++p) {
                s_row_off[g->w[j].rings[p]] = wi.send_off[j] + (int64_t)p;
                s_row_stride[g->w[j].rings[p]] = R[j];
            }
        for (int j = 0; j < W; ++j)
            for (size_t c = 0; c < g->w[j].ms.size(); ++c) s_m_base[g->w[j].ms[c]] = wi.recv_off[j] + (int64_t)c * R[i];
        // (SHTC_GROUP_RING_MAJOR=1 keeps the ring-major blocks: the comparison layout)
        static const bool ring_major = std::getenv("SHTC_GROUP_RING_MAJOR") && std::atoi(std::getenv("SHTC_GROUP_RING_MAJOR"));
        if (!ring_major)
            cck(shtc_set_exchange_layout_synthesis(wi.ctx, s_row_off.data(), s_row_stride.data(), s_m_base.data(),
                                                   s_m_stride.data()),
                wi, "exchange layout (synthesis)");
        if (g->mode == SHTC_EXCHANGE_PEER) {
            // store targets: ring r's element of worker i's first order in the ring owner's recv
            // block from i (order-major); order m's column (ring position 0) in the order
            // owner's send block for i (ring-major)
            std::vector<uint64_t> row_ptr(g->n_rings, 0), col_ptr(g->mmax + 1, 0);
            for (int j = 0; j < W; ++j) {
                const Worker& wj = g->w[j];
                for (size_t p = 0; p < wj.rings.size(); ++p)
                    row_ptr[wj.rings[p]] = (uint64_t)wj.recv +
                                           16ull * (uint64_t)(wj.recv_off[i] + (int64_t)p * (ring_major ? M[i] : 1));
                for (size_t c = 0; c < wj.ms.size(); ++c)
                    col_ptr[wj.ms[c]] = (uint64_t)wj.send + 16ull * (uint64_t)(wj.send_off[i] + (int64_t)c);
            }
            cck(shtc_set_exchange_peers(wi.ctx, row_ptr.data(), col_ptr.data()), wi, "exchange peers");
        }
    }
}

void sync_all(shtc_group* g) {
    for (Worker& w : g->w) {
        GCK(cudaSetDevice(w.dev));
        GCK(cudaStreamSynchronize(w.s));
    }
}

// every stream waits for every worker's completion of the previous call (its consumer stage
// read the buffers this call's producer stage stores into)
void order_after_previous(shtc_group* g) {
    if (!g->ran) return;
    for (Worker& w : g->w) {
        GCK(cudaSetDevice(w.dev));
        for (Worker& o : g->w) GCK(cudaStreamWaitEvent(w.s, o.ev[5], 0));
    }
}

// the exchange between stage 1 (events ev[2]) and stage 2
void exchange(shtc_group* g, bool to_rings) {
    if (g->mode == SHTC_EXCHANGE_PEER) {
        // the producers' stores are complete when their stage-1 events fire
        for (Worker& w : g->w) {
            GCK(cudaSetDevice(w.dev));
            for (Worker& o : g->w)
                if (&o != &w) GCK(cudaStreamWaitEvent(w.s, o.ev[2], 0));
        }
    } else {
        const Nccl& N = Nccl::get();
        const int W = (int)g->w.size();
        N.check(N.GroupStart(), "ncclGroupStart");
        for (int i = 0; i < W; ++i) {
            Worker& wi = g->w[i];
            // alm2map: send blocks (per ring owner) -> the owner's recv block from i;
            // map2alm: recv-shaped blocks (per order owner) -> the owner's send block from i
            auto* src = static_cast<double2*>(to_rings ? wi.send : wi.recv);
            auto* dst = static_cast<double2*>(to_rings ? wi.recv : wi.send);
            const auto& so = to_rings ? wi.send_off : wi.recv_off;
            const auto& sc = to_rings ? wi.send_cnt : wi.recv_cnt;
            const auto& ro = to_rings ? wi.recv_off : wi.send_off;
            const auto& rc = to_rings ? wi.recv_cnt : wi.send_cnt;
            for (int j = 0; j < W; ++j) {
                if (sc[j] > 0) N.check(N.Send(src + so[j], 2 * (size_t)sc[j], ncclDouble, j, wi.comm, wi.s), "ncclSend");
                if (rc[j] > 0) N.check(N.Recv(dst + ro[j], 2 * (size_t)rc[j], ncclDouble, j, wi.comm, wi.s), "ncclRecv");
            }
        }
        N.check(N.GroupEnd(), "ncclGroupEnd");
    }
    for (Worker& w : g->w) {
        GCK(cudaSetDevice(w.dev));
        GCK(cudaEventRecord(w.ev[3], w.s));
    }
}

void fill_gtiming(shtc_group* g, shtc_group_timing* t, bool synth, double wall_ms) {
    if (!t) return;
    *t = shtc_group_timing{};
    double leg = 0, fft = 0, xch = 0, h2d = 0, d2h = 0;
    for (Worker& w : g->w) {
        GCK(cudaSetDevice(w.dev));
        float e[kEv - 1];
        for (int k = 0; k + 1 < kEv; ++k) GCK(cudaEventElapsedTime(&e[k], w.ev[k], w.ev[k + 1]));
        h2d = std::max(h2d, (double)e[0]);
        (synth ? leg : fft) = std::max(synth ? leg : fft, (double)e[1]);
        xch = std::max(xch, (double)e[2]);
        (synth ? fft : leg) = std::max(synth ? fft : leg, (double)e[3]);
        d2h = std::max(d2h, (double)e[4]);
        t->nominal_steps += w.nominal;
    }
    t->legendre_ms = leg;
    t->fft_ms = fft;
    t->exchange_ms = xch;
    t->h2d_ms = h2d;
    t->d2h_ms = d2h;
    t->total_ms = wall_ms;
    const int W = (int)g->w.size();
    for (int i = 0; i < W; ++i)
        for (int j = 0; j < W; ++j)
            if (j != i) t->exchange_bytes += 16ull * (uint64_t)g->w[i].send_cnt[j];
}

void require_ready(shtc_group* g) {
    if (!g->grid_set) gfail(SHTC_EINVAL, "shtc_group: no grid set");
    if (!g->layout_set) gfail(SHTC_EINVAL, "shtc_group: no layout set");
}

// alm2map over the group.  host: alm / map are host buffers (H2D / D2H inside); else alm_dev /
// map_dev are per-worker device buffers (full triangle / full map on that worker's device).
void run_alm2map(shtc_group* g, const double* alm, double* map, const uint64_t* alm_dev, const uint64_t* map_dev,
                 shtc_group_timing* t) {
    require_ready(g);
    const auto t0 = std::chrono::steady_clock::now();
    const bool host = alm_dev == nullptr;
    const size_t na = alm_count(g->lmax, g->mmax);
    const double* src = alm;
    double* dst = map;
    bool stage_out = false;
    if (host) {
        if (!shtc_host::host_pinned(alm)) {
            g->stage_alm.ensure(na * 16);
            shtc_host::par_memcpy(g->stage_alm.p, alm, na * 16);
            src = static_cast<const double*>(g->stage_alm.p);
        }
        if (!shtc_host::host_pinned(map)) {
            g->stage_map.ensure((size_t)g->npix * 8);
            dst = static_cast<double*>(g->stage_map.p);
            stage_out = true;
        }
    }
    order_after_previous(g);
    for (size_t i = 0; i < g->w.size(); ++i) {
        Worker& w = g->w[i];
        GCK(cudaSetDevice(w.dev));
        GCK(cudaEventRecord(w.ev[0], w.s));
        const double* a = host ? static_cast<const double*>(w.a_dev) : reinterpret_cast<const double*>(alm_dev[i]);
        if (host) cck(shtc_copy_orders(w.ctx, src, static_cast<double*>(w.a_dev), 1), w, "a_lm H2D");
        GCK(cudaEventRecord(w.ev[1], w.s));
        if (g->mode == SHTC_EXCHANGE_PEER)
            cck(shtc_legendre_alm2map_peer(w.ctx, a, nullptr), w, "Legendre stage");
        else
            cck(shtc_legendre_alm2map_dev(w.ctx, a, static_cast<double*>(w.send), nullptr), w, "Legendre stage");
        GCK(cudaEventRecord(w.ev[2], w.s));
    }
    exchange(g, true);
    for (size_t i = 0; i < g->w.size(); ++i) {
        Worker& w = g->w[i];
        GCK(cudaSetDevice(w.dev));
        double* m = host ? static_cast<double*>(w.m_dev) : reinterpret_cast<double*>(map_dev[i]);
        cck(shtc_ring_synthesis_dev(w.ctx, static_cast<const double*>(w.recv), m, nullptr), w, "ring synthesis");
        GCK(cudaEventRecord(w.ev[4], w.s));
        if (host)
            for (const auto& iv : w.pix)
                GCK(cudaMemcpyAsync(dst + iv.first, m + iv.first, (size_t)(iv.second - iv.first) * 8,
                                    cudaMemcpyDeviceToHost, w.s));
        GCK(cudaEventRecord(w.ev[5], w.s));
    }
    g->ran = true;
    sync_all(g);
    if (stage_out) shtc_host::par_memcpy(map, dst, (size_t)g->npix * 8);
    const double wall = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    fill_gtiming(g, t, true, wall);
}

void run_map2alm(shtc_group* g, const double* map, double* alm, const uint64_t* map_dev, const uint64_t* alm_dev,
                 shtc_group_timing* t) {
    require_ready(g);
    const auto t0 = std::chrono::steady_clock::now();
    const bool host = map_dev == nullptr;
    const size_t na = alm_count(g->lmax, g->mmax);
    const double* src = map;
    double* dst = alm;
    bool stage_out = false;
    if (host) {
        if (!shtc_host::host_pinned(map)) {
            g->stage_map.ensure((size_t)g->npix * 8);
            shtc_host::par_memcpy(g->stage_map.p, map, (size_t)g->npix * 8);
            src = static_cast<const double*>(g->stage_map.p);
        }
        if (!shtc_host::host_pinned(alm)) {
            g->stage_alm.ensure(na * 16);
            dst = static_cast<double*>(g->stage_alm.p);
            stage_out = true;
        }
    }
    order_after_previous(g);
    for (size_t i = 0; i < g->w.size(); ++i) {
        Worker& w = g->w[i];
        GCK(cudaSetDevice(w.dev));
        GCK(cudaEventRecord(w.ev[0], w.s));
        const double* m = host ? static_cast<const double*>(w.m_dev) : reinterpret_cast<const double*>(map_dev[i]);
        if (host)
            for (const auto& iv : w.pix)
                GCK(cudaMemcpyAsync(static_cast<double*>(w.m_dev) + iv.first, src + iv.first,
                                    (size_t)(iv.second - iv.first) * 8, cudaMemcpyHostToDevice, w.s));
        GCK(cudaEventRecord(w.ev[1], w.s));
        if (g->mode == SHTC_EXCHANGE_PEER)
            cck(shtc_ring_analysis_peer(w.ctx, m, nullptr), w, "ring analysis");
        else
            cck(shtc_ring_analysis_dev(w.ctx, m, static_cast<double*>(w.recv), nullptr), w, "ring analysis");
        GCK(cudaEventRecord(w.ev[2], w.s));
    }
    exchange(g, false);
    for (size_t i = 0; i < g->w.size(); ++i) {
        Worker& w = g->w[i];
        GCK(cudaSetDevice(w.dev));
        double* a = host ? static_cast<double*>(w.a_dev) : reinterpret_cast<double*>(alm_dev[i]);
        cck(shtc_legendre_map2alm_dev(w.ctx, static_cast<const double*>(w.send), a, nullptr), w, "Legendre stage");
        GCK(cudaEventRecord(w.ev[4], w.s));
        if (host) cck(shtc_copy_orders(w.ctx, a, dst, 0), w, "a_lm D2H");
        GCK(cudaEventRecord(w.ev[5], w.s));
    }
    g->ran = true;
    sync_all(g);
    if (stage_out) shtc_host::par_memcpy(alm, dst, na * 16);
    const double wall = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    fill_gtiming(g, t, false, wall);
}

}  // namespace

extern "C" {

const char* shtc_group_last_error(const shtc_group* g) { return g ? g->err.c_str() : g_group_error.c_str(); }

shtc_status shtc_group_create(int n_workers, const int32_t* device_ids, int exchange_mode, shtc_group** out) {
    if (!out) return SHTC_EINVAL;
    *out = nullptr;
    return gguard(nullptr, [&] {
        if (n_workers < 1) gfail(SHTC_EINVAL, "shtc_group_create: n_workers must be >= 1");
        if (exchange_mode != SHTC_EXCHANGE_PEER && exchange_mode != SHTC_EXCHANGE_NCCL)
            gfail(SHTC_EINVAL, "shtc_group_create: unknown exchange mode");
        int nd = 0;
        GCK(cudaGetDeviceCount(&nd));
        auto g = std::make_unique<shtc_group>();
        g->mode = exchange_mode;
        g->w.resize(n_workers);
        std::vector<int> devs(n_workers);
        for (int i = 0; i < n_workers; ++i) {
            devs[i] = device_ids ? device_ids[i] : i % std::max(nd, 1);
            if (devs[i] < 0 || devs[i] >= nd) gfail(SHTC_EINVAL, "shtc_group_create: no such CUDA device");
        }
        // fused stores between distinct devices need peer access (NVLink / NVSwitch)
        for (int i = 0; i < n_workers; ++i)
            for (int j = 0; j < n_workers; ++j) {
                if (devs[i] == devs[j]) continue;
                int can = 0;
                GCK(cudaDeviceCanAccessPeer(&can, devs[i], devs[j]));
                if (!can) {
                    if (exchange_mode == SHTC_EXCHANGE_PEER)
                        gfail(SHTC_EUNSUPPORTED, "shtc_group_create: devices " + std::to_string(devs[i]) + " and " +
                                                     std::to_string(devs[j]) + " have no peer access");
                    continue;
                }
                GCK(cudaSetDevice(devs[i]));
                const cudaError_t e = cudaDeviceEnablePeerAccess(devs[j], 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                else GCK(e);
            }
        for (int i = 0; i < n_workers; ++i) {
            Worker& w = g->w[i];
            w.dev = devs[i];
            const shtc_status st = shtc_create(w.dev, &w.ctx);
            if (st != SHTC_OK) gfail(st, std::string("shtc_group_create: ") + shtc_last_error(nullptr));
            GCK(cudaSetDevice(w.dev));
            GCK(cudaStreamCreateWithFlags(&w.s, cudaStreamNonBlocking));
            for (auto& e : w.ev) GCK(cudaEventCreate(&e));
            cck(shtc_set_stream(w.ctx, w.s), w, "set stream");
        }
        if (exchange_mode == SHTC_EXCHANGE_NCCL) {
            std::vector<int> sorted = devs;
            std::sort(sorted.begin(), sorted.end());
            if (std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end())
                gfail(SHTC_EUNSUPPORTED, "shtc_group_create: the NCCL exchange needs one distinct device per worker");
            const Nccl& N = Nccl::get();
            if (!N.ok) gfail(SHTC_EUNSUPPORTED, "shtc_group_create: " + N.why);
            std::vector<ncclComm_t> comms(n_workers);
            N.check(N.CommInitAll(comms.data(), n_workers, devs.data()), "ncclCommInitAll");
            for (int i = 0; i < n_workers; ++i) g->w[i].comm = comms[i];
        }
        *out = g.release();
    });
}

void shtc_group_destroy(shtc_group* g) {
    if (!g) return;
    for (Worker& w : g->w) {
        cudaSetDevice(w.dev);
        if (w.s) cudaStreamSynchronize(w.s);
    }
    for (Worker& w : g->w) {
        if (w.comm) Nccl::get().CommDestroy(w.comm);
        free_buffers(w);
        if (w.ctx) shtc_destroy(w.ctx);
        cudaSetDevice(w.dev);
        for (auto& e : w.ev)
            if (e) cudaEventDestroy(e);
        if (w.s) cudaStreamDestroy(w.s);
    }
    delete g;
}

shtc_status shtc_group_device(const shtc_group* g, int worker, int* device) {
    if (!g || !device || worker < 0 || worker >= (int)g->w.size()) return SHTC_EINVAL;
    *device = g->w[worker].dev;
    return SHTC_OK;
}

shtc_status shtc_group_set_grid(shtc_group* g, int n_rings, const double* cos_theta, const int32_t* n_phi,
                                const double* phi_0, const double* weight, const int64_t* pixel_offset, int mirror) {
    if (!g) return SHTC_EINVAL;
    return gguard(g, [&] {
        for (Worker& w : g->w)
            cck(shtc_set_grid(w.ctx, n_rings, cos_theta, n_phi, phi_0, weight, pixel_offset, mirror), w, "set grid");
        g->n_rings = n_rings;
        g->cos_theta.assign(cos_theta, cos_theta + n_rings);
        g->nphi.assign(n_phi, n_phi + n_rings);
        g->phi0.assign(phi_0, phi_0 + n_rings);
        g->weight.assign(weight, weight + n_rings);
        g->pixoff.resize(n_rings);
        int64_t off = 0;
        for (int r = 0; r < n_rings; ++r) {
            g->pixoff[r] = pixel_offset ? pixel_offset[r] : off;
            off += n_phi[r];
        }
        g->npix = off;
        g->mirror = mirror;
        g->grid_set = true;
        g->layout_set = false;
    });
}

shtc_status shtc_group_set_layout(shtc_group* g, int lmax, int mmax, const int32_t* m_owner,
                                  const int32_t* ring_owner) {
    if (!g || !m_owner || !ring_owner) return SHTC_EINVAL;
    return gguard(g, [&] {
        if (!g->grid_set) gfail(SHTC_EINVAL, "shtc_group: no grid set");
        if (lmax < mmax || mmax < 0) gfail(SHTC_EINVAL, "analysis: need lmax >= mmax >= 0");
        const int W = (int)g->w.size();
        sync_all(g);
        g->layout_set = false;
        g->ran = false;
        for (Worker& w : g->w) {
            w.ms.clear();
            w.rings.clear();
            w.pix.clear();
        }
        for (int m = 0; m <= mmax; ++m) {
            if (m_owner[m] < 0 || m_owner[m] >= W) gfail(SHTC_EINVAL, "shtc_group: order owner out of range");
            g->w[m_owner[m]].ms.push_back(m);
        }
        for (int r = 0; r < g->n_rings; ++r) {
            if (ring_owner[r] < 0 || ring_owner[r] >= W) gfail(SHTC_EINVAL, "exchange: invalid ring layout");
            Worker& w = g->w[ring_owner[r]];
            w.rings.push_back(r);
            const int64_t b = g->pixoff[r], e = b + g->nphi[r];
            if (!w.pix.empty() && w.pix.back().second == b) w.pix.back().second = e;
            else w.pix.push_back({b, e});
        }
        for (int i = 0; i < W; ++i)
            if (g->w[i].ms.empty() || g->w[i].rings.empty())
                gfail(SHTC_EINVAL, "shtc_group: worker " + std::to_string(i) +
                                       " owns no order or no ring (assign_m / assign_rings never do that)");
        g->lmax = lmax;
        g->mmax = mmax;
        const auto t0 = std::chrono::steady_clock::now();
        for (Worker& w : g->w) {
            GCK(cudaSetDevice(w.dev));
            cck(shtc_set_band(w.ctx, lmax, mmax, (int)w.ms.size(), w.ms.data()), w, "set band");
        }
        build_exchange(g);
        // build every Legendre plan now (the ring plans come with the exchange layout)
        for (Worker& w : g->w) {
            uint64_t nominal = 0;
            cck(shtc_plan_stats(w.ctx, &nominal, nullptr, nullptr), w, "plan");
            w.nominal = nominal;
        }
        sync_all(g);
        g->plan_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        g->layout_set = true;
    });
}

shtc_status shtc_group_plan_ms(const shtc_group* g, double* plan_ms) {
    if (!g || !plan_ms) return SHTC_EINVAL;
    *plan_ms = g->plan_ms;
    return SHTC_OK;
}

shtc_status shtc_group_alm2map(shtc_group* g, const double* alm, double* map, shtc_group_timing* t) {
    if (!g || !alm || !map) return SHTC_EINVAL;
    return gguard(g, [&] { run_alm2map(g, alm, map, nullptr, nullptr, t); });
}

shtc_status shtc_group_map2alm(shtc_group* g, const double* map, double* alm, shtc_group_timing* t) {
    if (!g || !alm || !map) return SHTC_EINVAL;
    return gguard(g, [&] { run_map2alm(g, map, alm, nullptr, nullptr, t); });
}

shtc_status shtc_group_alm2map_dev(shtc_group* g, const uint64_t* alm_dev, const uint64_t* map_dev,
                                   shtc_group_timing* t) {
    if (!g || !alm_dev || !map_dev) return SHTC_EINVAL;
    return gguard(g, [&] { run_alm2map(g, nullptr, nullptr, alm_dev, map_dev, t); });
}

shtc_status shtc_group_map2alm_dev(shtc_group* g, const uint64_t* map_dev, const uint64_t* alm_dev,
                                   shtc_group_timing* t) {
    if (!g || !alm_dev || !map_dev) return SHTC_EINVAL;
    return gguard(g, [&] { run_map2alm(g, nullptr, nullptr, map_dev, alm_dev, t); });
}

}  // extern "C"
