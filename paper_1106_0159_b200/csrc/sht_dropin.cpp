// libsht_b200: the reference's C++ API (namespace sht, include/sht/*.hpp) as a drop-in over
// the C ABI (include/shtc.h).  Host side only: validation with the reference's error classes,
// containers, geometry, layouts and step accounting; every transform runs on the GPU.
//
// Reference behaviour mirrored (file:line in /root/reference/proj):
//   grid builders                 src/grid.cpp:23-151
//   AlmSet                        src/alm.cpp:7-16
//   synthesis / analysis          src/transforms.cpp:402-485 (checks :403, :448-455)
//   Legendre-stage operators      src/transforms.cpp:222-400 (checked_m_set, check_latitudes,
//                                 accumulate_core, reduce_partials)
//   layouts, exchange, drivers    src/distribution.cpp:53-490
//   Profiler                      src/perfmodel.cpp:57-83
//   inputs                        src/experiment.cpp:11-44
// The GPU context is process-wide and created on first use (the reference API has no
// handle); calls are serialised by a mutex.  SHT_DEVICE selects the CUDA device.

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <mutex>
#include <numbers>
#include <numeric>
#include <stdexcept>
#include <string>
#include <thread>

#include "sht/alm.hpp"
#include "sht/distribution.hpp"
#include "sht/experiment.hpp"
#include "sht/grid.hpp"
#include "sht/legendre.hpp"
#include "sht/perfmodel.hpp"
#include "sht/transforms.hpp"
#include "shtc.h"
#include "hostcopy.h"

namespace sht {

namespace {

constexpr double kPi = std::numbers::pi;

[[noreturn]] void raise(shtc_status st, const shtc_ctx* c) {
    const std::string msg = shtc_last_error(c);
    switch (st) {
        case SHTC_EINVAL: throw std::invalid_argument(msg);
        case SHTC_EDOMAIN: throw std::domain_error(msg);
        default: throw std::runtime_error("sht (B200): " + msg);
    }
}

void ok(shtc_status st, const shtc_ctx* c) {
    if (st != SHTC_OK) raise(st, c);
}

struct GridKey {
    std::vector<double> cos, phi0, w;
    std::vector<int> nphi;
    int mirror = -1;
    bool operator==(const GridKey&) const = default;
};

GridKey grid_key(const PixelGrid& g, bool mirror) {
    GridKey k;
    for (const auto& r : g.rings) {
        k.cos.push_back(r.cos_theta);
        k.phi0.push_back(r.phi_0);
        k.w.push_back(r.weight);
        k.nphi.push_back(r.n_phi);
    }
    k.mirror = mirror ? 1 : 0;
    return k;
}

std::vector<int64_t> pixel_offsets(const PixelGrid& g) {
    std::vector<int64_t> off;
    for (const auto& r : g.rings) off.push_back(r.pixel_offset);
    return off;
}

// Devices of an n-worker group: SHT_DEVICES="0,1,..." (worker i on entry i mod its length), else
// worker i on device i mod the device count (workers share a device on smaller boxes)
std::vector<int32_t> worker_devices(int n) {
    std::vector<int32_t> list;
    if (const char* e = std::getenv("SHT_DEVICES")) {
        for (const char* q = e; *q;) {
            list.push_back(std::atoi(q));
            while (*q && *q != ',') ++q;
            if (*q) ++q;
        }
    }
    if (list.empty()) {
        const int nd = std::max(1, shtc_device_count());
        for (int i = 0; i < nd; ++i) list.push_back(i);
    }
    std::vector<int32_t> d(n);
    for (int i = 0; i < n; ++i) d[i] = list[i % list.size()];
    return d;
}

[[noreturn]] void raise_group(shtc_status st, const shtc_group* g) {
    const std::string msg = shtc_group_last_error(g);
    switch (st) {
        case SHTC_EINVAL: throw std::invalid_argument(msg);
        case SHTC_EDOMAIN: throw std::domain_error(msg);
        default: throw std::runtime_error("sht (B200): " + msg);
    }
}

void gok(shtc_status st, const shtc_group* g) {
    if (st != SHTC_OK) raise_group(st, g);
}

struct Engine {
    std::mutex mu;
    shtc_ctx* ctx = nullptr;
    GridKey grid;
    int lmax = -1, mmax = -1;
    bool ladder = true;
    // multi-worker layouts: one shtc_group (W device contexts) per worker count in use
    shtc_group* grp = nullptr;
    int grp_workers = 0;
    GridKey grp_grid;
    int grp_lmax = -1, grp_mmax = -1;
    std::vector<std::vector<int>> grp_msets, grp_rsets;

    // page-locked result buffer (grows, kept for the process): large transforms write their
    // output here while the returned container is value-initialised on a helper thread
    void* pin = nullptr;
    size_t pin_bytes = 0;
    double* pinned(size_t bytes) {
        if (bytes > pin_bytes) {
            shtc_host_free(pin);
            pin = nullptr;
            pin_bytes = 0;
            if (shtc_host_alloc(bytes, &pin) != SHTC_OK) throw std::runtime_error("sht: page-locked allocation failed");
            pin_bytes = bytes;
        }
        return static_cast<double*>(pin);
    }

    shtc_ctx* get() {
        if (!ctx) {
            const char* d = std::getenv("SHT_DEVICE");
            ok(shtc_create(d ? std::atoi(d) : 0, &ctx), nullptr);
        }
        return ctx;
    }
    void bind(const PixelGrid& g, int lmax_, int mmax_, bool mirror) {
        shtc_ctx* c = get();
        GridKey k = grid_key(g, mirror);
        if (!(k == grid)) {
            std::vector<int32_t> np32(k.nphi.begin(), k.nphi.end());
            const auto off = pixel_offsets(g);
            ok(shtc_set_grid(c, (int)k.cos.size(), k.cos.data(), np32.data(), k.phi0.data(), k.w.data(), off.data(),
                             mirror ? 1 : 0),
               c);
            grid = std::move(k);
            lmax = mmax = -1;
        }
        if (lmax != lmax_ || mmax != mmax_) {
            ok(shtc_set_band(c, lmax_, mmax_, 0, nullptr), c);
            lmax = lmax_;
            mmax = mmax_;
        }
    }
    void set_ladder(const ScaleLadder& l) {
        // the GPU plans know the reference's two ladders; any other window is refused
        const bool standard = l.enabled && l.step == 0x1p512 && l.inv_step == 0x1p-512 && l.hi == 0x1p512 &&
                              l.lo == 0x1p-512;
        if (l.enabled && !standard)
            throw std::invalid_argument("ScaleLadder: only ScaleLadder::standard() and ScaleLadder::unscaled() "
                                        "are supported by the GPU plans");
        shtc_ctx* c = get();
        if (ladder != l.enabled) {
            ok(shtc_set_ladder(c, l.enabled ? 1 : 0), c);
            ladder = l.enabled;
        }
    }
    shtc_group* group(const PixelGrid& g, const WorkerLayout& l, int lmax_, int mmax_, bool mirror) {
        const int W = l.n_workers;
        if (grp && grp_workers != W) {
            shtc_group_destroy(grp);
            grp = nullptr;
        }
        if (!grp) {
            const char* ex = std::getenv("SHT_EXCHANGE");
            const int mode = (ex && std::string(ex) == "nccl") ? SHTC_EXCHANGE_NCCL : SHTC_EXCHANGE_PEER;
            const auto devs = worker_devices(W);
            gok(shtc_group_create(W, devs.data(), mode, &grp), nullptr);
            grp_workers = W;
            grp_grid = GridKey{};
            grp_msets.clear();
        }
        GridKey k = grid_key(g, mirror);
        if (!(k == grp_grid)) {
            std::vector<int32_t> np32(k.nphi.begin(), k.nphi.end());
            const auto off = pixel_offsets(g);
            gok(shtc_group_set_grid(grp, (int)k.cos.size(), k.cos.data(), np32.data(), k.phi0.data(), k.w.data(),
                                    off.data(), mirror ? 1 : 0),
                grp);
            grp_grid = std::move(k);
            grp_msets.clear();
        }
        if (grp_msets != l.m_sets || grp_rsets != l.ring_sets || grp_lmax != lmax_ || grp_mmax != mmax_) {
            std::vector<int32_t> mo(mmax_ + 1), ro(g.n_rings());
            for (int w = 0; w < W; ++w) {
                for (int m : l.m_sets[w]) mo[m] = w;
                for (int r : l.ring_sets[w]) ro[r] = w;
            }
            gok(shtc_group_set_layout(grp, lmax_, mmax_, mo.data(), ro.data()), grp);
            grp_msets = l.m_sets;
            grp_rsets = l.ring_sets;
            grp_lmax = lmax_;
            grp_mmax = mmax_;
        }
        return grp;
    }
};

// The reference API returns its results by value in value-initialised std::vectors.  For a
// large result the zero fill (page faults on one thread: 147-160 ms for the 403 MB C4 map) costs
// far more than the transform, so it runs on a helper thread (huge-page advice + parallel first
// touch + memset, shtc_host::value_init) while the GPU transform writes into the engine's
// page-locked buffer; the result is then copied in on all host cores with streaming stores.
template <class T, class Xform>
void into_container(Engine& e, std::vector<T>& v, size_t n, Xform&& xform) {
    const size_t bytes = n * sizeof(T);
    if (bytes < (size_t(16) << 20)) {
        v.assign(n, T{});
        xform(reinterpret_cast<double*>(v.data()));
        return;
    }
    double* out = e.pinned(bytes);
    std::exception_ptr fill_err;
    std::thread filler([&] {
        try {
            shtc_host::value_init(v, n);
        } catch (...) {
            fill_err = std::current_exception();
        }
    });
    try {
        xform(out);
    } catch (...) {
        filler.join();
        throw;
    }
    filler.join();
    if (fill_err) std::rethrow_exception(fill_err);
    shtc_host::par_memcpy(v.data(), out, bytes);
}

Engine& engine() {
    static Engine e;
    return e;
}

std::vector<int> checked_m_set(std::span<const int> m_set, int mmax, const char* where) {
    std::vector<int> ms(m_set.begin(), m_set.end());
    std::sort(ms.begin(), ms.end());
    for (size_t i = 0; i < ms.size(); ++i) {
        if (ms[i] < 0 || ms[i] > mmax)
            throw std::invalid_argument(std::string(where) + ": order outside [0, mmax]");
        if (i > 0 && ms[i] == ms[i - 1])
            throw std::invalid_argument(std::string(where) + ": duplicate order");
    }
    return ms;
}

void check_latitudes(std::span<const double> x, const char* where) {
    for (double v : x)
        if (!(std::fabs(v) <= 1.0))
            throw std::invalid_argument(std::string(where) + ": cos_theta outside [-1, 1]");
}

std::vector<int> iota_n(size_t n) {
    std::vector<int> r(n);
    std::iota(r.begin(), r.end(), 0);
    return r;
}

uint64_t order_steps(int lmax, const std::vector<int>& ms) {
    uint64_t s = 0;
    for (int m : ms) s += (uint64_t)(lmax - m + 1);
    return s;
}

}  // namespace

// ---- legendre parameters ----------------------------------------------------------------
const ScaleLadder& ScaleLadder::standard() {
    static const ScaleLadder l{};
    return l;
}
const ScaleLadder& ScaleLadder::unscaled() {
    static const ScaleLadder l = [] {
        ScaleLadder s;
        s.enabled = false;
        return s;
    }();
    return l;
}

double log_mu(int m) {
    if (m < 0) throw std::invalid_argument("log_mu: m must be >= 0");
    return -m * std::numbers::ln2 - std::lgamma(m + 1.0) +
           0.5 * (std::lgamma(2.0 * m + 2.0) - 2.5310242469692907930);
}

double beta_lm(int l, int m) {
    if (m < 0 || l < m) throw std::invalid_argument("beta_lm: need l >= m >= 0");
    if (l == m) throw std::domain_error("beta_lm: undefined at l == m");
    const double dl = l, dm = m;
    return std::sqrt((4.0 * dl * dl - 1.0) / (dl * dl - dm * dm));
}

// ---- containers and geometry -------------------------------------------------------------
AlmSet::AlmSet(int lmax_, int mmax_) : lmax(lmax_), mmax(mmax_) {
    if (lmax < 0 || mmax < 0 || mmax > lmax)
        throw std::invalid_argument("AlmSet: need lmax >= mmax >= 0");
    values.assign(count(lmax, mmax), cdouble{0.0, 0.0});
}

std::size_t AlmSet::count(int lmax, int mmax) {
    const std::size_t l = lmax, m = mmax;
    return (m + 1) * (l + 1) - m * (m + 1) / 2;
}

std::vector<double> PixelGrid::cos_thetas() const {
    std::vector<double> z;
    z.reserve(rings.size());
    for (const auto& r : rings) z.push_back(r.cos_theta);
    return z;
}

PixelGrid build_healpix_grid(int nside) {
    if (nside < 1) throw std::invalid_argument("healpix grid: nside must be >= 1");
    PixelGrid g;
    g.scheme = GridScheme::healpix_ring;
    g.nside = nside;
    g.n_pix = 12LL * nside * nside;
    const int nr = 4 * nside - 1;
    g.rings.resize(nr);
    const double w = 4.0 * kPi / static_cast<double>(g.n_pix);
    for (int i = 1; i <= 2 * nside; ++i) {
        RingDescriptor& r = g.rings[i - 1];
        if (i < nside) {
            r.n_phi = 4 * i;
            r.cos_theta = 1.0 - static_cast<double>(i) * i / (3.0 * nside * nside);
            r.phi_0 = kPi / (4.0 * i);
        } else {
            r.n_phi = 4 * nside;
            r.cos_theta = 4.0 / 3.0 - 2.0 * i / (3.0 * nside);
            r.phi_0 = ((i - nside) % 2 == 0) ? kPi / (4.0 * nside) : 0.0;
        }
        r.sin_theta = std::sqrt((1.0 - r.cos_theta) * (1.0 + r.cos_theta));
        r.weight = w;
    }
    for (int i = 2 * nside + 1; i <= nr; ++i) {
        g.rings[i - 1] = g.rings[(4 * nside - i) - 1];
        g.rings[i - 1].cos_theta = -g.rings[i - 1].cos_theta;
    }
    std::int64_t off = 0;
    for (int k = 0; k < nr; ++k) {
        g.rings[k].index = k;
        g.rings[k].pixel_offset = off;
        off += g.rings[k].n_phi;
    }
    if (off != g.n_pix) throw std::runtime_error("healpix grid: pixel count mismatch");
    return g;
}

std::pair<std::vector<double>, std::vector<double>> gauss_legendre_nodes(int n) {
    if (n < 1) throw std::invalid_argument("gauss_legendre_nodes: n must be >= 1");
    std::vector<double> x(n), w(n);
    for (int i = 0; i < (n + 1) / 2; ++i) {
        double t = std::cos(kPi * (i + 0.75) / (n + 0.5)), dp = 0.0;
        bool done = false;
        for (int it = 0; it < 100 && !done; ++it) {
            double p0 = 1.0, p1 = t;
            for (int l = 2; l <= n; ++l) {
                const double p2 = ((2.0 * l - 1.0) * t * p1 - (l - 1.0) * p0) / l;
                p0 = p1;
                p1 = p2;
            }
            dp = n * (p0 - t * p1) / (1.0 - t * t);
            const double dt = p1 / dp;
            t -= dt;
            done = std::abs(dt) < 1e-15;
        }
        if (!done) throw std::runtime_error("gauss_legendre_nodes: Newton iteration failed");
        x[i] = t;
        w[i] = 2.0 / ((1.0 - t * t) * dp * dp);
        x[n - 1 - i] = -t;
        w[n - 1 - i] = w[i];
    }
    if (n % 2 == 1) x[n / 2] = 0.0;
    return {x, w};
}

PixelGrid build_gauss_legendre_grid(int n_rings, int n_phi) {
    if (n_rings < 1) throw std::invalid_argument("gauss-legendre grid: n_rings must be >= 1");
    if (n_phi < 1) throw std::invalid_argument("gauss-legendre grid: n_phi must be >= 1");
    auto [x, glw] = gauss_legendre_nodes(n_rings);
    PixelGrid g;
    g.scheme = GridScheme::gauss_legendre;
    g.n_pix = static_cast<std::int64_t>(n_rings) * n_phi;
    g.rings.resize(n_rings);
    for (int k = 0; k < n_rings; ++k) {
        RingDescriptor& r = g.rings[k];
        r.index = k;
        r.cos_theta = x[k];
        r.sin_theta = std::sqrt((1.0 - x[k]) * (1.0 + x[k]));
        r.n_phi = n_phi;
        r.weight = 2.0 * kPi / n_phi * glw[k];
        r.pixel_offset = static_cast<std::int64_t>(k) * n_phi;
    }
    return g;
}

std::vector<std::pair<int, std::optional<int>>> symmetric_ring_pairs(const PixelGrid& g) {
    const int n = g.n_rings();
    std::vector<std::pair<int, std::optional<int>>> out;
    for (int k = 0; k < n / 2; ++k) {
        const auto &a = g.rings[k], &b = g.rings[n - 1 - k];
        if (a.n_phi != b.n_phi || std::abs(a.cos_theta + b.cos_theta) > 1e-14)
            throw std::invalid_argument("symmetric_ring_pairs: grid is not mirror symmetric");
        out.emplace_back(k, n - 1 - k);
    }
    if (n % 2 == 1) {
        if (std::abs(g.rings[n / 2].cos_theta) > 1e-14)
            throw std::invalid_argument("symmetric_ring_pairs: central ring is off the equator");
        out.emplace_back(n / 2, std::nullopt);
    }
    return out;
}

std::string to_string(GridScheme s) {
    return s == GridScheme::healpix_ring ? "healpix-ring" : "gauss-legendre";
}

// ---- Legendre-stage operators --------------------------------------------------------------
namespace {
DeltaPanel delta_panel(const AlmSet& alm, std::span<const double> x, std::span<const int> m_set,
                       const ScaleLadder& ladder, std::uint64_t* steps, const char* where) {
    auto ms = checked_m_set(m_set, alm.mmax, where);
    check_latitudes(x, where);
    DeltaPanel p;
    p.kind = DeltaKind::synthesis;
    p.rings = iota_n(x.size());
    p.ms = ms;
    p.entries.assign(x.size() * ms.size(), cdouble{0.0, 0.0});
    Engine& e = engine();
    std::lock_guard<std::mutex> lock(e.mu);
    shtc_ctx* c = e.get();
    e.set_ladder(ladder);
    std::vector<int32_t> ms32(ms.begin(), ms.end());
    ok(shtc_delta_a(c, reinterpret_cast<const double*>(alm.values.data()), alm.lmax, alm.mmax,
                    (int)x.size(), x.data(), (int)ms32.size(), ms32.data(),
                    reinterpret_cast<double*>(p.entries.data()), steps),
       c);
    return p;
}

AlmSet accumulate_core(const DeltaPanel& panel, std::span<const double> x, int lmax, int mmax,
                       const ScaleLadder& ladder, std::uint64_t* steps, const char* where) {
    if (lmax < mmax || mmax < 0) throw std::invalid_argument(std::string(where) + ": need lmax >= mmax >= 0");
    if (x.size() != panel.rings.size())
        throw std::invalid_argument(std::string(where) + ": latitude count != panel rings");
    check_latitudes(x, where);
    for (int m : panel.ms)
        if (m < 0 || m > mmax) throw std::invalid_argument(std::string(where) + ": panel order outside [0, mmax]");
    AlmSet out(lmax, mmax);
    const size_t nr = panel.rings.size(), nc = panel.ms.size();
    if (nr == 0 || nc == 0) {
        if (steps) *steps += order_steps(lmax, panel.ms) * nr;
        return out;
    }
    // the C ABI takes ascending unique orders: permute columns; a repeated order (allowed by
    // the reference, whose columns simply add) becomes an extra call accumulating into out
    std::vector<size_t> idx(nc);
    std::iota(idx.begin(), idx.end(), 0);
    std::stable_sort(idx.begin(), idx.end(), [&](size_t a, size_t b) { return panel.ms[a] < panel.ms[b]; });
    std::vector<std::vector<size_t>> groups;
    for (size_t k = 0; k < nc; ++k) {
        size_t g = 0;
        while (g < groups.size() && !groups[g].empty() &&
               panel.ms[groups[g].back()] == panel.ms[idx[k]])
            ++g;
        if (g == groups.size()) groups.emplace_back();
        groups[g].push_back(idx[k]);
    }
    Engine& e = engine();
    std::lock_guard<std::mutex> lock(e.mu);
    shtc_ctx* c = e.get();
    e.set_ladder(ladder);
    for (const auto& cols : groups) {
        std::vector<int32_t> ms32;
        std::vector<cdouble> sub(nr * cols.size());
        for (size_t j = 0; j < cols.size(); ++j) {
            ms32.push_back(panel.ms[cols[j]]);
            for (size_t r = 0; r < nr; ++r) sub[r * cols.size() + j] = panel.entries[r * nc + cols[j]];
        }
        ok(shtc_accumulate_alm(c, reinterpret_cast<const double*>(sub.data()), (int)nr, x.data(),
                               (int)ms32.size(), ms32.data(), lmax, mmax,
                               reinterpret_cast<double*>(out.values.data()), steps),
           c);
    }
    return out;
}
}  // namespace

DeltaPanel compute_delta_a(const AlmSet& alm, std::span<const double> cos_thetas,
                           std::span<const int> m_set, const ScaleLadder& ladder, std::uint64_t* step_counter) {
    return delta_panel(alm, cos_thetas, m_set, ladder, step_counter, "compute_delta_a");
}

DeltaPanel compute_delta_a_ring_major(const AlmSet& alm, std::span<const double> cos_thetas,
                                      std::span<const int> m_set, int n_work_items, const ScaleLadder& ladder,
                                      std::uint64_t* step_counter) {
    if (n_work_items < 1)
        throw std::invalid_argument("compute_delta_a_ring_major: n_work_items must be >= 1");
    return delta_panel(alm, cos_thetas, m_set, ladder, step_counter, "compute_delta_a_ring_major");
}

AlmSet accumulate_alm(const DeltaPanel& panel, std::span<const double> cos_thetas, int lmax, int mmax,
                      const ScaleLadder& ladder, std::uint64_t* step_counter) {
    for (size_t i = 0; i < panel.rings.size(); ++i)
        if (panel.rings[i] != static_cast<int>(i))
            throw std::invalid_argument("accumulate_alm: ring coverage incomplete");
    return accumulate_core(panel, cos_thetas, lmax, mmax, ladder, step_counter, "accumulate_alm");
}

PartialAlm accumulate_alm_partial(const DeltaPanel& panel, std::span<const double> cos_thetas, int lmax,
                                  int mmax, const ScaleLadder& ladder, std::uint64_t* step_counter) {
    for (size_t i = 1; i < panel.rings.size(); ++i)
        if (panel.rings[i] <= panel.rings[i - 1])
            throw std::invalid_argument("accumulate_alm_partial: rings not strictly ascending");
    PartialAlm p;
    p.alm = accumulate_core(panel, cos_thetas, lmax, mmax, ladder, step_counter, "accumulate_alm_partial");
    p.rings = panel.rings;
    return p;
}

AlmSet reduce_partials(std::span<const PartialAlm> parts, std::size_t n_rings) {
    if (parts.empty()) throw std::invalid_argument("reduce_partials: no partials");
    const int lmax = parts[0].alm.lmax, mmax = parts[0].alm.mmax;
    std::vector<int> seen;
    for (const auto& p : parts) {
        if (p.alm.lmax != lmax || p.alm.mmax != mmax)
            throw std::invalid_argument("reduce_partials: mismatched band limits");
        seen.insert(seen.end(), p.rings.begin(), p.rings.end());
    }
    std::sort(seen.begin(), seen.end());
    for (size_t i = 1; i < seen.size(); ++i)
        if (seen[i] == seen[i - 1]) throw std::invalid_argument("reduce_partials: overlapping ring subsets");
    if (seen.size() != n_rings || (n_rings > 0 && (seen.front() != 0 || seen.back() != (int)n_rings - 1)))
        throw std::invalid_argument("reduce_partials: ring subsets do not cover the grid");
    AlmSet out(lmax, mmax);
    for (const auto& p : parts)
        for (size_t i = 0; i < out.values.size(); ++i) out.values[i] += p.alm.values[i];
    return out;
}

// ---- whole transforms ------------------------------------------------------------------------
namespace {
uint64_t streams_of(const PixelGrid& g, PairPolicy pp) {
    return pp == PairPolicy::mirror ? (uint64_t)(g.n_rings() + 1) / 2 : (uint64_t)g.n_rings();
}

using Clock = std::chrono::steady_clock;
double seconds_since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

// PairPolicy::mirror runs one stream per mirror ring pair (delta_a_columns_paired,
// transforms.cpp:145-182) and needs a mirror-symmetric grid; PairPolicy::none one stream per
// ring (delta_a_columns, :53-72)
void check_grid(const PixelGrid& grid, PairPolicy pairing, const char* where) {
    if (grid.n_rings() == 0) throw std::invalid_argument(std::string(where) + ": empty grid");
    check_latitudes(grid.cos_thetas(), where);
    if (pairing == PairPolicy::mirror) (void)symmetric_ring_pairs(grid);
}

// binds the grid / band and builds the plan; returns the host-visible precompute seconds
// (the reference's log_mu table + mirror pairs, here the GPU plan when it is (re)built)
double bind_planned(Engine& e, const PixelGrid& grid, int lmax, int mmax, PairPolicy pairing) {
    const auto t0 = Clock::now();
    e.set_ladder(ScaleLadder::standard());
    e.bind(grid, lmax, mmax, pairing == PairPolicy::mirror);
    ok(shtc_plan(e.ctx, nullptr), e.ctx);
    return seconds_since(t0);
}

SkyMap run_synthesis(const AlmSet& alm, const PixelGrid& grid, PairPolicy pairing, shtc_timing* t,
                     double* precompute_s = nullptr) {
    check_grid(grid, pairing, "synthesis");
    SkyMap map;
    map.grid = grid;
    Engine& e = engine();
    std::lock_guard<std::mutex> lock(e.mu);
    const double pre = bind_planned(e, grid, alm.lmax, alm.mmax, pairing);
    if (precompute_s) *precompute_s = pre;
    into_container(e, map.pixels, static_cast<size_t>(grid.n_pix), [&](double* out) {
        ok(shtc_alm2map(e.ctx, reinterpret_cast<const double*>(alm.values.data()), out, t), e.ctx);
    });
    return map;
}

AlmSet run_analysis(const SkyMap& map, int lmax, int mmax, PairPolicy pairing, shtc_timing* t,
                    double* precompute_s = nullptr) {
    if (lmax < mmax || mmax < 0) throw std::invalid_argument("analysis: need lmax >= mmax >= 0");
    const PixelGrid& grid = map.grid;
    if (grid.n_rings() == 0) throw std::invalid_argument("analysis: empty grid");
    if (map.pixels.size() != static_cast<size_t>(grid.n_pix))
        throw std::invalid_argument("analysis: pixel count != grid");
    check_grid(grid, pairing, "analysis");
    AlmSet out;
    out.lmax = lmax;
    out.mmax = mmax;
    Engine& e = engine();
    std::lock_guard<std::mutex> lock(e.mu);
    const double pre = bind_planned(e, grid, lmax, mmax, pairing);
    if (precompute_s) *precompute_s = pre;
    into_container(e, out.values, AlmSet::count(lmax, mmax), [&](double* dst) {
        ok(shtc_map2alm(e.ctx, map.pixels.data(), dst, t), e.ctx);
    });
    return out;
}
}  // namespace

SkyMap synthesis(const AlmSet& alm, const PixelGrid& grid, const TransformOptions& o) {
    SkyMap m = run_synthesis(alm, grid, o.pairing, nullptr);
    if (o.step_counter)
        *o.step_counter += streams_of(grid, o.pairing) * order_steps(alm.lmax, iota_n(alm.mmax + 1));
    return m;
}

AlmSet analysis(const SkyMap& map, int lmax, int mmax, const TransformOptions& o) {
    AlmSet a = run_analysis(map, lmax, mmax, o.pairing, nullptr);
    if (o.step_counter)
        *o.step_counter += streams_of(map.grid, o.pairing) * order_steps(lmax, iota_n(mmax + 1));
    return a;
}

// ---- distribution -----------------------------------------------------------------------------
std::vector<std::vector<int>> assign_m(int mmax, int n_workers) {
    if (mmax < 0) throw std::invalid_argument("assign_m: mmax must be >= 0");
    if (n_workers < 1) throw std::invalid_argument("assign_m: n_workers must be >= 1");
    if (n_workers > 1 && n_workers > (mmax + 1) / 2) throw std::invalid_argument("assign_m: n_workers > mmax/2");
    std::vector<std::vector<int>> sets(n_workers);
    int lo = 0, hi = mmax, w = 0;
    for (; lo < hi; ++lo, --hi, w = (w + 1) % n_workers) {
        sets[w].push_back(lo);
        sets[w].push_back(hi);
    }
    if (lo == hi) sets[w].push_back(lo);
    for (auto& s : sets) std::sort(s.begin(), s.end());
    return sets;
}

std::vector<std::vector<int>> assign_rings(const PixelGrid& grid, int n_workers) {
    const int rn = grid.n_rings();
    if (n_workers < 1) throw std::invalid_argument("assign_rings: n_workers must be >= 1");
    if (rn < 1) throw std::invalid_argument("assign_rings: empty grid");
    if (n_workers == 1) return {iota_n(rn)};
    if (2 * n_workers > rn) throw std::invalid_argument("assign_rings: n_workers > n_rings/2");
    const int h = (rn + 1) / 2, q = h / n_workers, rem = h % n_workers;
    std::vector<std::vector<int>> sets(n_workers);
    for (int w = 0, row = 0; w < n_workers; ++w) {
        for (int j = 0; j < q + (w < rem ? 1 : 0); ++j, ++row) {
            sets[w].push_back(row);
            if (rn - 1 - row != row) sets[w].push_back(rn - 1 - row);
        }
        std::sort(sets[w].begin(), sets[w].end());
    }
    return sets;
}

std::vector<std::vector<int>> thread_partition(const std::vector<int>& m_set, int n_threads) {
    if (n_threads <= 0) throw std::invalid_argument("thread_partition: n_threads must be >= 1");
    std::vector<int> ms = m_set;
    std::sort(ms.begin(), ms.end());
    std::vector<std::vector<int>> sets(n_threads);
    if (ms.empty()) return sets;
    const long long top = ms.back();
    std::vector<long long> load(n_threads, 0);
    size_t lo = 0, hi = ms.size() - 1;
    int t = 0;
    for (; lo < hi; ++lo, --hi, t = (t + 1) % n_threads) {
        sets[t].push_back(ms[lo]);
        sets[t].push_back(ms[hi]);
        load[t] += (top + 1 - ms[lo]) + (top + 1 - ms[hi]);
    }
    if (lo == hi) sets[std::min_element(load.begin(), load.end()) - load.begin()].push_back(ms[lo]);
    for (auto& s : sets) std::sort(s.begin(), s.end());
    return sets;
}

WorkerLayout WorkerLayout::create(const PixelGrid& grid, int mmax, int n_workers) {
    WorkerLayout l;
    l.n_workers = n_workers;
    l.mmax = mmax;
    l.n_rings = grid.n_rings();
    l.m_sets = n_workers == 1 ? std::vector<std::vector<int>>{iota_n(mmax + 1)} : assign_m(mmax, n_workers);
    l.ring_sets = assign_rings(grid, n_workers);
    return l;
}

std::uint64_t ExchangeVolume::total() const {
    std::uint64_t t = 0;
    for (const auto& row : bytes)
        for (auto b : row) t += b;
    return t;
}

namespace {
void check_exchange(const std::vector<DeltaPanel>& panels, const WorkerLayout& l, bool m_sliced, const char* where) {
    if (panels.size() != static_cast<size_t>(l.n_workers))
        throw std::invalid_argument(std::string(where) + ": panel count != n_workers");
    for (int i = 0; i < l.n_workers; ++i) {
        const DeltaPanel& p = panels[i];
        const bool shape = m_sliced ? (p.ms == l.m_sets[i] && p.rings == iota_n(l.n_rings))
                                    : (p.rings == l.ring_sets[i] && p.ms == iota_n(l.mmax + 1));
        if (!shape) throw std::invalid_argument(std::string(where) + ": layout mismatch");
        if (p.entries.size() != p.rings.size() * p.ms.size())
            throw std::invalid_argument(std::string(where) + ": panel shape mismatch");
    }
}
}  // namespace

std::vector<DeltaPanel> exchange_m_to_rings(const std::vector<DeltaPanel>& panels, const WorkerLayout& l,
                                            ExchangeVolume* volume) {
    check_exchange(panels, l, true, "exchange_m_to_rings");
    const int nw = l.n_workers;
    const size_t nm = static_cast<size_t>(l.mmax) + 1;
    std::vector<std::pair<int, size_t>> owner(l.n_rings, {-1, 0});
    for (int w = 0; w < nw; ++w)
        for (size_t j = 0; j < l.ring_sets[w].size(); ++j) owner[l.ring_sets[w][j]] = {w, j};
    std::vector<DeltaPanel> out(nw);
    for (int w = 0; w < nw; ++w) {
        out[w].kind = panels[0].kind;
        out[w].rings = l.ring_sets[w];
        out[w].ms = iota_n(nm);
        out[w].entries.assign(out[w].rings.size() * nm, cdouble{});
    }
    if (volume) volume->bytes.assign(nw, std::vector<std::uint64_t>(nw, 0));
    for (int s = 0; s < nw; ++s)
        for (int r = 0; r < l.n_rings; ++r) {
            auto [w, j] = owner[r];
            for (size_t c = 0; c < panels[s].ms.size(); ++c)
                out[w].entries[j * nm + panels[s].ms[c]] = panels[s].entries[r * panels[s].ms.size() + c];
            if (volume) volume->bytes[s][w] += panels[s].ms.size() * 16;
        }
    return out;
}

std::vector<DeltaPanel> exchange_rings_to_m(const std::vector<DeltaPanel>& panels, const WorkerLayout& l,
                                            ExchangeVolume* volume) {
    check_exchange(panels, l, false, "exchange_rings_to_m");
    const int nw = l.n_workers;
    const size_t nm = static_cast<size_t>(l.mmax) + 1;
    std::vector<DeltaPanel> out(nw);
    for (int w = 0; w < nw; ++w) {
        out[w].kind = panels[0].kind;
        out[w].rings = iota_n(l.n_rings);
        out[w].ms = l.m_sets[w];
        out[w].entries.assign(l.n_rings * out[w].ms.size(), cdouble{});
    }
    if (volume) volume->bytes.assign(nw, std::vector<std::uint64_t>(nw, 0));
    for (int s = 0; s < nw; ++s)
        for (size_t j = 0; j < panels[s].rings.size(); ++j) {
            const size_t r = panels[s].rings[j];
            for (int d = 0; d < nw; ++d) {
                const auto& ms = out[d].ms;
                for (size_t c = 0; c < ms.size(); ++c) out[d].entries[r * ms.size() + c] = panels[s].entries[j * nm + ms[c]];
                if (volume) volume->bytes[s][d] += ms.size() * 16;
            }
        }
    return out;
}

namespace {
void check_layout(const WorkerLayout& l, const PixelGrid& g, int mmax, const RunOptions& o, const char* where) {
    if (l.n_workers < 1 || l.m_sets.size() != static_cast<size_t>(l.n_workers) ||
        l.ring_sets.size() != static_cast<size_t>(l.n_workers))
        throw std::invalid_argument(std::string(where) + ": malformed layout");
    if (l.n_rings != g.n_rings()) throw std::invalid_argument(std::string(where) + ": layout built for another grid");
    if (l.mmax != mmax) throw std::invalid_argument(std::string(where) + ": layout built for another mmax");
    if (o.n_threads < 1) throw std::invalid_argument(std::string(where) + ": n_threads must be >= 1");
    if (o.pairing == PairPolicy::mirror && o.kernel == KernelOrder::ring_major)
        throw std::invalid_argument(std::string(where) + ": mirror pairing needs the m-major kernel");
}

// The ownership the drivers run: ring_sets must cover every ring exactly once, with the
// reference exchange's own errors (ring_owners, distribution.cpp:215-228); m_sets must
// partition 0..mmax (the reference leaves out-of-range orders undefined and sums overlapping
// ones; the GPU drivers refuse both).
void check_ownership(const WorkerLayout& l, const char* where) {
    std::vector<int> ring_owner(l.n_rings, -1);
    for (int w = 0; w < l.n_workers; ++w)
        for (int r : l.ring_sets[w]) {
            if (r < 0 || r >= l.n_rings || ring_owner[r] >= 0) throw std::invalid_argument("exchange: invalid ring layout");
            ring_owner[r] = w;
        }
    for (int o : ring_owner)
        if (o < 0) throw std::invalid_argument("exchange: ring layout gap");
    std::vector<int> m_owner(l.mmax + 1, -1);
    for (int w = 0; w < l.n_workers; ++w)
        for (int m : l.m_sets[w]) {
            if (m < 0 || m > l.mmax) throw std::invalid_argument(std::string(where) + ": order outside [0, mmax]");
            if (m_owner[m] >= 0) throw std::invalid_argument(std::string(where) + ": order owned by two workers");
            m_owner[m] = w;
        }
    for (int o : m_owner)
        if (o < 0) throw std::invalid_argument(std::string(where) + ": m_sets do not cover 0..mmax");
}

// The reference's per-(worker, thread) nominal step slots (distribution.cpp:324-347) and stage
// seconds (:313, :349, :355, :377): precompute = plan (re)build on the host API path, recurrence
// = the Legendre stage, exchange = the Delta transpose (the wait between the stages on the fused
// path, the NCCL time on the NCCL path; 0 with one worker), fft = the ring stage.
void fill_profiler(Profiler* prof, const WorkerLayout& l, const PixelGrid& g, int lmax, const RunOptions& o,
                   double precompute_s, double leg_ms, double fft_ms, double exchange_ms) {
    if (!prof) return;
    prof->configure(l.n_workers, o.n_threads);
    const uint64_t streams = streams_of(g, o.pairing);
    for (int w = 0; w < l.n_workers; ++w) {
        if (o.kernel == KernelOrder::ring_major) {
            const size_t nr = g.n_rings();
            for (int th = 0; th < o.n_threads; ++th) {
                const size_t b = nr * th / o.n_threads, e = nr * (th + 1) / o.n_threads;
                *prof->step_slot(w, th) += (e - b) * order_steps(lmax, l.m_sets[w]);
            }
        } else {
            auto parts = thread_partition(l.m_sets[w], o.n_threads);
            for (int th = 0; th < o.n_threads; ++th) *prof->step_slot(w, th) += streams * order_steps(lmax, parts[th]);
        }
    }
    prof->precompute_s += precompute_s;
    prof->recurrence_s += leg_ms * 1e-3;
    prof->fft_s += fft_ms * 1e-3;
    prof->exchange_s += exchange_ms * 1e-3;
    // ExchangeVolume::total of the reference transpose: every Delta entry once (self blocks too)
    prof->exchange_bytes += (uint64_t)g.n_rings() * (l.mmax + 1) * 16;
}
}  // namespace

SkyMap distributed_synthesis(const AlmSet& alm, const PixelGrid& grid, const WorkerLayout& layout,
                             const RunOptions& o) {
    check_layout(layout, grid, alm.mmax, o, "distributed_synthesis");
    check_ownership(layout, "distributed_synthesis");
    if (layout.n_workers == 1) {
        shtc_timing t{};
        double pre = 0.0;
        SkyMap m = run_synthesis(alm, grid, o.pairing, &t, &pre);
        fill_profiler(o.profiler, layout, grid, alm.lmax, o, pre, t.legendre_ms, t.fft_ms, 0.0);
        return m;
    }
    // W workers = W device contexts (worker i on device i mod the device count, or SHT_DEVICES)
    check_grid(grid, o.pairing, "distributed_synthesis");
    SkyMap map;
    map.grid = grid;
    shtc_group_timing t{};
    double pre = 0.0;
    {
        Engine& e = engine();
        std::lock_guard<std::mutex> lock(e.mu);
        const auto t0 = Clock::now();
        shtc_group* g = e.group(grid, layout, alm.lmax, alm.mmax, o.pairing == PairPolicy::mirror);
        pre = seconds_since(t0);
        into_container(e, map.pixels, static_cast<size_t>(grid.n_pix), [&](double* out) {
            gok(shtc_group_alm2map(g, reinterpret_cast<const double*>(alm.values.data()), out, &t), g);
        });
    }
    fill_profiler(o.profiler, layout, grid, alm.lmax, o, pre, t.legendre_ms, t.fft_ms, t.exchange_ms);
    return map;
}

AlmSet distributed_analysis(const SkyMap& map, int lmax, int mmax, const WorkerLayout& layout,
                            const RunOptions& o) {
    if (lmax < mmax || mmax < 0) throw std::invalid_argument("distributed_analysis: need lmax >= mmax >= 0");
    if (map.pixels.size() != static_cast<size_t>(map.grid.n_pix))
        throw std::invalid_argument("distributed_analysis: pixel count != grid");
    check_layout(layout, map.grid, mmax, o, "distributed_analysis");
    check_ownership(layout, "distributed_analysis");
    if (layout.n_workers == 1) {
        shtc_timing t{};
        double pre = 0.0;
        AlmSet a = run_analysis(map, lmax, mmax, o.pairing, &t, &pre);
        fill_profiler(o.profiler, layout, map.grid, lmax, o, pre, t.legendre_ms, t.fft_ms, 0.0);
        return a;
    }
    check_grid(map.grid, o.pairing, "distributed_analysis");
    AlmSet out;
    out.lmax = lmax;
    out.mmax = mmax;
    shtc_group_timing t{};
    double pre = 0.0;
    {
        Engine& e = engine();
        std::lock_guard<std::mutex> lock(e.mu);
        const auto t0 = Clock::now();
        shtc_group* g = e.group(map.grid, layout, lmax, mmax, o.pairing == PairPolicy::mirror);
        pre = seconds_since(t0);
        into_container(e, out.values, AlmSet::count(lmax, mmax), [&](double* dst) {
            gok(shtc_group_map2alm(g, map.pixels.data(), dst, &t), g);
        });
    }
    fill_profiler(o.profiler, layout, map.grid, lmax, o, pre, t.legendre_ms, t.fft_ms, t.exchange_ms);
    return out;
}

// ---- Profiler -----------------------------------------------------------------------------------
void Profiler::configure(int n_workers, int n_threads) {
    if (n_workers < 1 || n_threads < 1)
        throw std::invalid_argument("Profiler: worker and thread counts must be >= 1");
    n_workers_ = n_workers;
    n_threads_ = n_threads;
    steps_.assign(static_cast<size_t>(n_workers) * n_threads, 0);
    precompute_s = recurrence_s = exchange_s = fft_s = 0.0;
    exchange_bytes = 0;
}
std::uint64_t* Profiler::step_slot(int w, int t) {
    if (w < 0 || w >= n_workers_ || t < 0 || t >= n_threads_) throw std::out_of_range("Profiler::step_slot");
    return &steps_[static_cast<size_t>(w) * n_threads_ + t];
}
std::uint64_t Profiler::slot_steps(int w, int t) const {
    if (w < 0 || w >= n_workers_ || t < 0 || t >= n_threads_) throw std::out_of_range("Profiler::slot_steps");
    return steps_[static_cast<size_t>(w) * n_threads_ + t];
}
std::uint64_t Profiler::total_steps() const { return std::accumulate(steps_.begin(), steps_.end(), std::uint64_t{0}); }

// ---- inputs -------------------------------------------------------------------------------------
std::uint64_t splitmix64_at(std::uint64_t seed, std::uint64_t index) {
    std::uint64_t z = seed + (index + 1) * 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

double uniform_pm1(std::uint64_t seed, std::uint64_t index) {
    return 2.0 * ((static_cast<double>(splitmix64_at(seed, index) >> 11) + 0.5) * 0x1p-53) - 1.0;
}

AlmSet random_alm(int lmax, int mmax, std::uint64_t seed) {
    AlmSet a(lmax, mmax);
    for (size_t k = 0; k < a.values.size(); ++k) a.values[k] = {uniform_pm1(seed, 2 * k), uniform_pm1(seed, 2 * k + 1)};
    for (int l = 0; l <= lmax; ++l) a.at(l, 0).imag(0.0);
    return a;
}

double roundtrip_error(const AlmSet& a, const AlmSet& b) {
    if (a.lmax != b.lmax || a.mmax != b.mmax) throw std::invalid_argument("roundtrip_error: mismatched band limits");
    double num = 0.0, den = 0.0;
    for (size_t i = 0; i < a.values.size(); ++i) {
        num += std::norm(a.values[i] - b.values[i]);
        den += std::norm(a.values[i]);
    }
    if (den == 0.0) throw std::domain_error("roundtrip_error: zero reference norm");
    return std::sqrt(num / den);
}

}  // namespace sht
