// C++ parity suite of the drop-in API (include/sht/*.hpp, libsht_b200.so -> libshtc.so, GPU)
// against the reference itself (oracle/_ref/libsht_ref.so through its C shim).  Restates the
// reference's own unit tests (test_transforms.cpp, test_distribution.cpp) on the GPU path.
// Built and run by tests/test_gpu_cpp.py; prints "PASS n" / "FAIL ..." lines.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "sht/distribution.hpp"
#include "sht/experiment.hpp"
#include "sht/grid.hpp"
#include "sht/transforms.hpp"

extern "C" {
int ref_synthesis(int, int, const double*, int, int, int, const double*, const int32_t*, const double*,
                  const double*, int, int, double*, uint64_t*);
int ref_analysis(int, int, const double*, int, int, int, const double*, const int32_t*, const double*,
                 const double*, int, double*, uint64_t*);
int ref_compute_delta_a(int, int, const double*, int, const double*, int, const int32_t*, int, int, int,
                        double*, uint64_t*);
int ref_accumulate_alm(int, int, int, const double*, int, const int32_t*, const double*, double*, uint64_t*);
int ref_distributed_synthesis(int, int, const double*, int, int, int, const double*, const int32_t*,
                              const double*, const double*, int, int, int, int, double*, double*, uint64_t*);
int ref_distributed_analysis(int, int, const double*, int, int, int, const double*, const int32_t*,
                             const double*, const double*, int, int, int, int, double*, double*, uint64_t*);
}

static int fails = 0, passes = 0;
#define CHECK(cond, what)                                                        \
    do {                                                                         \
        if (cond) ++passes;                                                      \
        else { ++fails; std::printf("FAIL %s (line %d)\n", what, __LINE__); }    \
    } while (0)

using sht::cdouble;

static sht::AlmSet make_random_alm(int lmax, int mmax, unsigned seed) {
    std::mt19937 gen(seed);
    std::uniform_real_distribution<double> d(-1.0, 1.0);
    sht::AlmSet a(lmax, mmax);
    for (auto& v : a.values) v = cdouble{d(gen), d(gen)};
    for (int l = 0; l <= lmax; ++l) a.at(l, 0).imag(0.0);
    return a;
}

struct RefGrid {
    std::vector<double> c, p, w;
    std::vector<int32_t> n;
    explicit RefGrid(const sht::PixelGrid& g) {
        for (auto& r : g.rings) { c.push_back(r.cos_theta); p.push_back(r.phi_0); w.push_back(r.weight); n.push_back(r.n_phi); }
    }
};

static double rel_rms(const double* a, const double* b, size_t n) {
    double num = 0, den = 0;
    for (size_t i = 0; i < n; ++i) { num += (a[i] - b[i]) * (a[i] - b[i]); den += b[i] * b[i]; }
    return std::sqrt(num / (den > 0 ? den : 1));
}

int main() {
    const double kY00 = 0.28209479177387814;
    // monopole -> constant map (test_transforms.cpp:70-80)
    {
        sht::AlmSet alm(8, 8);
        alm.at(0, 0) = cdouble{3.25, 0.0};
        for (const auto& g : {sht::build_healpix_grid(4), sht::build_gauss_legendre_grid(9, 20)}) {
            auto m = sht::synthesis(alm, g);
            double worst = 0;
            for (double p : m.pixels) worst = std::max(worst, std::fabs(p - 3.25 * kY00));
            CHECK(worst <= 1e-14 * 3.25 * kY00 * 10, "monopole synthesis");
        }
    }
    // analysis of a constant map on a quadrature grid (test_transforms.cpp:82-97)
    {
        auto g = sht::build_gauss_legendre_grid(33, 66);
        sht::SkyMap m;
        m.grid = g;
        m.pixels.assign(g.n_pix, -1.7);
        auto a = sht::analysis(m, 32, 32);
        CHECK(std::fabs(a.at(0, 0).real() - (-1.7 / kY00)) <= 1e-13 * 1.7 / kY00, "constant map monopole");
        double stray = 0;
        for (size_t i = 1; i < a.values.size(); ++i) stray = std::max(stray, std::abs(a.values[i]));
        CHECK(stray <= 1e-12 * 1.7 / kY00, "constant map stray");
    }
    // HEALPix synthesis / analysis against the reference (C1 and small grids)
    for (auto [ns, lmax] : std::vector<std::pair<int, int>>{{4, 12}, {16, 40}, {128, 256}}) {
        auto g = sht::build_healpix_grid(ns);
        auto alm = sht::random_alm(lmax, lmax, 12345);
        RefGrid rg(g);
        std::vector<double> want(g.n_pix);
        uint64_t steps = 0;
        ref_synthesis(lmax, lmax, reinterpret_cast<const double*>(alm.values.data()), 0, ns, g.n_rings(),
                      rg.c.data(), rg.n.data(), rg.p.data(), rg.w.data(), 1, 0, want.data(), &steps);
        sht::TransformOptions opt;
        opt.pairing = sht::PairPolicy::mirror;
        uint64_t mysteps = 0;
        opt.step_counter = &mysteps;
        auto m = sht::synthesis(alm, g, opt);
        CHECK(rel_rms(m.pixels.data(), want.data(), want.size()) <= 1e-12, "healpix synthesis vs reference");
        CHECK(mysteps == steps, "synthesis step counter");
        std::vector<double> aw(2 * alm.values.size());
        ref_analysis(lmax, lmax, want.data(), 0, ns, g.n_rings(), rg.c.data(), rg.n.data(), rg.p.data(),
                     rg.w.data(), 1, aw.data(), &steps);
        sht::SkyMap in{g, want};
        auto a = sht::analysis(in, lmax, lmax, opt);
        CHECK(rel_rms(reinterpret_cast<const double*>(a.values.data()), aw.data(), aw.size()) <= 1e-12,
              "healpix analysis vs reference");
    }
    // C2 (nside 1024, lmax 2048): results above the drop-in's large-container threshold, which
    // are value-initialised on a helper thread while the GPU writes a page-locked buffer
    {
        const int ns = 1024, lmax = 2048;
        auto g = sht::build_healpix_grid(ns);
        auto alm = sht::random_alm(lmax, lmax, 2026);
        RefGrid rg(g);
        const int nt = (int)std::max(1u, std::thread::hardware_concurrency());
        std::vector<double> want(g.n_pix);
        ref_distributed_synthesis(lmax, lmax, reinterpret_cast<const double*>(alm.values.data()), 0, ns, g.n_rings(),
                                  rg.c.data(), rg.n.data(), rg.p.data(), rg.w.data(), 1, nt, 1, 0, want.data(),
                                  nullptr, nullptr);
        sht::TransformOptions opt;
        opt.pairing = sht::PairPolicy::mirror;
        auto m = sht::synthesis(alm, g, opt);
        CHECK(m.pixels.size() == want.size() && rel_rms(m.pixels.data(), want.data(), want.size()) <= 1e-10,
              "C2 synthesis (large result container) vs reference");
        std::vector<double> aw(2 * alm.values.size());
        ref_distributed_analysis(lmax, lmax, want.data(), 0, ns, g.n_rings(), rg.c.data(), rg.n.data(), rg.p.data(),
                                 rg.w.data(), 1, nt, 1, 0, aw.data(), nullptr, nullptr);
        sht::SkyMap in{g, want};
        auto a = sht::analysis(in, lmax, lmax, opt);
        CHECK(a.lmax == lmax && a.mmax == lmax && a.values.size() == alm.values.size() &&
                  rel_rms(reinterpret_cast<const double*>(a.values.data()), aw.data(), aw.size()) <= 1e-10,
              "C2 analysis (large result container) vs reference");
        // twice more: the page-locked buffer is reused and every call returns its own container
        auto m2 = sht::synthesis(alm, g, opt);
        CHECK(m2.pixels == m.pixels, "repeated C2 synthesis identical");
        auto lay = sht::WorkerLayout::create(g, lmax, 2);
        sht::RunOptions ro;
        ro.pairing = sht::PairPolicy::mirror;
        auto md = sht::distributed_synthesis(alm, g, lay, ro);
        CHECK(md.pixels == m.pixels, "C2 distributed synthesis (2 workers) = synthesis");
        auto ad = sht::distributed_analysis(in, lmax, lmax, lay, ro);
        CHECK(rel_rms(reinterpret_cast<const double*>(ad.values.data()), aw.data(), aw.size()) <= 1e-10,
              "C2 distributed analysis (2 workers) vs reference");
    }
    // delta panel and accumulation vs the reference (test_transforms.cpp:99-148)
    {
        auto [x, w] = sht::gauss_legendre_nodes(17);
        auto alm = make_random_alm(16, 16, 555);
        std::vector<int> ms(17);
        std::iota(ms.begin(), ms.end(), 0);
        uint64_t steps = 0, rsteps = 0;
        auto p = sht::compute_delta_a(alm, x, ms, sht::ScaleLadder::standard(), &steps);
        std::vector<double> want(2 * 17 * 17);
        std::vector<int32_t> ms32(ms.begin(), ms.end());
        ref_compute_delta_a(16, 16, reinterpret_cast<const double*>(alm.values.data()), 17, x.data(), 17,
                            ms32.data(), 0, 1, 0, want.data(), &rsteps);
        CHECK(rel_rms(reinterpret_cast<const double*>(p.entries.data()), want.data(), want.size()) <= 1e-13,
              "delta panel vs reference");
        CHECK(steps == rsteps, "delta step counter");
        auto pr = sht::compute_delta_a_ring_major(alm, x, ms, 3);
        CHECK(pr.entries == p.entries, "ring-major operator = m-major operator");
        std::mt19937 gen(808);
        std::uniform_real_distribution<double> d(-1.0, 1.0);
        sht::DeltaPanel dp;
        dp.kind = sht::DeltaKind::analysis;
        dp.rings.resize(17);
        std::iota(dp.rings.begin(), dp.rings.end(), 0);
        dp.ms = ms;
        dp.entries.resize(17 * 17);
        for (auto& e : dp.entries) e = cdouble{d(gen), d(gen)};
        auto acc = sht::accumulate_alm(dp, x, 16, 16);
        std::vector<double> wacc(2 * acc.values.size());
        ref_accumulate_alm(16, 16, 17, x.data(), 17, ms32.data(), reinterpret_cast<const double*>(dp.entries.data()),
                           wacc.data(), &rsteps);
        CHECK(rel_rms(reinterpret_cast<const double*>(acc.values.data()), wacc.data(), wacc.size()) <= 1e-13,
              "accumulate vs reference");
        // partial accumulations reduce to the full one (test_transforms.cpp:169-245)
        auto slice = [&](int lo, int hi) {
            sht::DeltaPanel s;
            s.kind = sht::DeltaKind::analysis;
            s.ms = ms;
            for (int r = lo; r < hi; ++r) {
                s.rings.push_back(r);
                for (size_t c = 0; c < ms.size(); ++c) s.entries.push_back(dp.at(r, c));
            }
            return s;
        };
        std::vector<sht::PartialAlm> parts;
        parts.push_back(sht::accumulate_alm_partial(slice(0, 9), std::vector<double>(x.begin(), x.begin() + 9), 16, 16));
        parts.push_back(sht::accumulate_alm_partial(slice(9, 17), std::vector<double>(x.begin() + 9, x.end()), 16, 16));
        auto red = sht::reduce_partials(parts, 17);
        CHECK(rel_rms(reinterpret_cast<const double*>(red.values.data()), wacc.data(), wacc.size()) <= 1e-13,
              "partials reduce to the full accumulation");
        bool threw = false;
        try { (void)sht::reduce_partials(std::vector<sht::PartialAlm>{parts[0]}, 17); } catch (const std::invalid_argument&) { threw = true; }
        CHECK(threw, "gap in coverage rejected");
    }
    // exact round trip on a quadrature grid (test_transforms.cpp:283-290)
    {
        auto g = sht::build_gauss_legendre_grid(33, 66);
        auto alm = make_random_alm(32, 32, 4242);
        auto back = sht::analysis(sht::synthesis(alm, g), 32, 32);
        CHECK(sht::roundtrip_error(alm, back) <= 1e-13, "GL round trip");
    }
    // distributed drivers: worker/thread invariance and profiler slots (test_distribution.cpp:256-352).
    // W > 1 runs W device contexts (shtc_group: worker i on device i mod the device count),
    // the Delta exchange as fused peer stores; synthesis is bitwise worker invariant, analysis
    // sums each order's ring partials in the same kernels (<= 1e-14 of the one-worker result)
    {
        auto g = sht::build_gauss_legendre_grid(128, 256);
        auto alm = make_random_alm(127, 127, 2024);
        auto ref_map = sht::synthesis(alm, g);
        auto ref_alm = sht::analysis(ref_map, 127, 127);
        for (int n : {1, 2, 3, 4, 8})
            for (int t : {1, 4}) {
                sht::RunOptions o;
                o.n_threads = t;
                auto layout = sht::WorkerLayout::create(g, 127, n);
                auto m = sht::distributed_synthesis(alm, g, layout, o);
                CHECK(m.pixels == ref_map.pixels, "distributed synthesis worker invariance");
                auto a = sht::distributed_analysis(ref_map, 127, 127, layout, o);
                CHECK(rel_rms(reinterpret_cast<const double*>(a.values.data()),
                              reinterpret_cast<const double*>(ref_alm.values.data()), 2 * a.values.size()) <= 1e-14,
                      "distributed analysis worker invariance");
            }
        sht::Profiler prof;
        sht::RunOptions o;
        o.n_threads = 2;
        o.profiler = &prof;
        (void)sht::distributed_synthesis(alm, g, sht::WorkerLayout::create(g, 127, 4), o);
        uint64_t want = 0;
        for (int m = 0; m <= 127; ++m) want += (uint64_t)g.n_rings() * (127 - m + 1);
        CHECK(prof.total_steps() == want, "profiler total steps");
        CHECK(prof.recurrence_s > 0 && prof.fft_s > 0 && prof.exchange_s >= 0 && prof.precompute_s >= 0,
              "profiler stage seconds");
        CHECK(prof.exchange_bytes == (uint64_t)g.n_rings() * 128 * 16, "profiler exchange bytes");
        // a new layout (W = 3) rebuilds the plans: the precompute stage is timed
        sht::Profiler prof3;
        o.profiler = &prof3;
        (void)sht::distributed_analysis(ref_map, 127, 127, sht::WorkerLayout::create(g, 127, 3), o);
        CHECK(prof3.precompute_s > 0 && prof3.recurrence_s > 0, "profiler precompute on a plan rebuild");
        sht::RunOptions bad;
        bad.kernel = sht::KernelOrder::ring_major;
        bad.pairing = sht::PairPolicy::mirror;
        bool threw = false;
        try { (void)sht::distributed_synthesis(alm, g, sht::WorkerLayout::create(g, 127, 2), bad); } catch (const std::invalid_argument&) { threw = true; }
        CHECK(threw, "mirror + ring_major rejected");
    }
    // distributed drivers against the reference at HEALPix nside 64 / lmax 128, mirror pairing,
    // W = 1, 2, 4, 8 workers (distribution.cpp:300-490 run by the reference with the same layout)
    {
        const int ns = 64, lmax = 128;
        auto g = sht::build_healpix_grid(ns);
        auto alm = sht::random_alm(lmax, lmax, 12345);
        RefGrid rg(g);
        std::vector<double> want(g.n_pix);
        uint64_t steps = 0;
        ref_synthesis(lmax, lmax, reinterpret_cast<const double*>(alm.values.data()), 0, ns, g.n_rings(),
                      rg.c.data(), rg.n.data(), rg.p.data(), rg.w.data(), 1, 0, want.data(), &steps);
        std::vector<double> aw(2 * alm.values.size());
        ref_analysis(lmax, lmax, want.data(), 0, ns, g.n_rings(), rg.c.data(), rg.n.data(), rg.p.data(),
                     rg.w.data(), 1, aw.data(), &steps);
        sht::SkyMap in{g, want};
        for (int n : {1, 2, 4, 8}) {
            sht::RunOptions o;
            o.pairing = sht::PairPolicy::mirror;
            auto layout = sht::WorkerLayout::create(g, lmax, n);
            auto m = sht::distributed_synthesis(alm, g, layout, o);
            CHECK(rel_rms(m.pixels.data(), want.data(), want.size()) <= 1e-12, "distributed synthesis vs reference");
            auto a = sht::distributed_analysis(in, lmax, lmax, layout, o);
            CHECK(rel_rms(reinterpret_cast<const double*>(a.values.data()), aw.data(), aw.size()) <= 1e-12,
                  "distributed analysis vs reference");
        }
        // layouts the reference's exchange refuses (ring_owners, distribution.cpp:215-228)
        auto layout = sht::WorkerLayout::create(g, lmax, 2);
        auto overlap = layout;
        overlap.ring_sets[1].push_back(overlap.ring_sets[0][0]);
        auto gap = layout;
        gap.ring_sets[1].pop_back();
        auto m_dup = layout;
        m_dup.m_sets[1].push_back(m_dup.m_sets[0][0]);
        std::string e1, e2;
        int n = 0;
        try { (void)sht::distributed_synthesis(alm, g, overlap); } catch (const std::invalid_argument& e) { e1 = e.what(); ++n; }
        try { (void)sht::distributed_analysis(in, lmax, lmax, gap); } catch (const std::invalid_argument& e) { e2 = e.what(); ++n; }
        try { (void)sht::distributed_synthesis(alm, g, m_dup); } catch (const std::invalid_argument&) { ++n; }
        CHECK(n == 3 && e1 == "exchange: invalid ring layout" && e2 == "exchange: ring layout gap",
              "distributed layout errors");
    }
    // mirror pairing reproduces the unpaired transforms (test_transforms.cpp:364-388); the
    // default PairPolicy::none runs unpaired streams, matching the reference's unpaired path
    for (auto [g, lmax] : std::vector<std::pair<sht::PixelGrid, int>>{{sht::build_healpix_grid(8), 20},
                                                                      {sht::build_gauss_legendre_grid(10, 24), 9}}) {
        auto alm = make_random_alm(lmax, lmax, 77);
        sht::TransformOptions paired;
        paired.pairing = sht::PairPolicy::mirror;
        auto plain_map = sht::synthesis(alm, g);
        auto paired_map = sht::synthesis(alm, g, paired);
        double worst = 0, peak = 0;
        for (size_t i = 0; i < plain_map.pixels.size(); ++i) {
            worst = std::max(worst, std::fabs(plain_map.pixels[i] - paired_map.pixels[i]));
            peak = std::max(peak, std::fabs(plain_map.pixels[i]));
        }
        CHECK(worst <= 1e-12 * std::max(1.0, peak), "mirror vs unpaired synthesis");
        auto plain_alm = sht::analysis(plain_map, lmax, lmax);
        auto paired_alm = sht::analysis(plain_map, lmax, lmax, paired);
        CHECK(rel_rms(reinterpret_cast<const double*>(paired_alm.values.data()),
                      reinterpret_cast<const double*>(plain_alm.values.data()), 2 * plain_alm.values.size()) <= 1e-12,
              "mirror vs unpaired analysis");
        RefGrid rg(g);
        std::vector<double> want(g.n_pix);
        uint64_t steps = 0;
        ref_synthesis(lmax, lmax, reinterpret_cast<const double*>(alm.values.data()), g.scheme == sht::GridScheme::healpix_ring ? 0 : 1,
                      g.nside, g.n_rings(), rg.c.data(), rg.n.data(), rg.p.data(), rg.w.data(), 0, 0, want.data(), &steps);
        CHECK(rel_rms(plain_map.pixels.data(), want.data(), want.size()) <= 1e-13, "unpaired synthesis vs reference");
    }
    // ScaleLadder::unscaled (test_transforms.cpp:150-167): identical panels where no stream
    // leaves the window; where a seed lies below it (m = 1500 at x = 0.5, P_mm ~ 2^-305) the
    // standard ladder activates the stream later, the unscaled one never counts it, exactly as
    // the reference's
    {
        auto [x, w] = sht::gauss_legendre_nodes(41);
        auto alm = make_random_alm(40, 40, 91);
        std::vector<int> ms(41);
        std::iota(ms.begin(), ms.end(), 0);
        auto by_m = sht::compute_delta_a(alm, x, ms);
        auto unscaled = sht::compute_delta_a(alm, x, ms, sht::ScaleLadder::unscaled());
        CHECK(unscaled.entries == by_m.entries, "unscaled ladder: identical panels");
        const int m = 1500, lmax = 2200;
        sht::AlmSet deep(lmax, lmax);
        std::mt19937 gen(5);
        std::normal_distribution<double> nd;
        for (int l = m; l <= lmax; ++l) deep.at(l, m) = cdouble{nd(gen), 0.0};
        const std::vector<double> xs{0.5, 0.3, 0.0, 0.6, -0.5};
        const std::vector<int> one{m};
        std::vector<int32_t> one32{m};
        for (bool uns : {false, true}) {
            auto got = sht::compute_delta_a(deep, xs, one, uns ? sht::ScaleLadder::unscaled() : sht::ScaleLadder::standard());
            std::vector<double> want(2 * xs.size());
            uint64_t st = 0;
            ref_compute_delta_a(lmax, lmax, reinterpret_cast<const double*>(deep.values.data()), (int)xs.size(), xs.data(), 1,
                                one32.data(), 0, 1, uns ? 1 : 0, want.data(), &st);
            double worst = 0, peak = 0;
            for (size_t i = 0; i < want.size(); ++i) {
                worst = std::max(worst, std::fabs(reinterpret_cast<const double*>(got.entries.data())[i] - want[i]));
                peak = std::max(peak, std::fabs(want[i]));
            }
            CHECK(worst <= 1e-10 * std::max(peak, 1e-300), uns ? "unscaled deep order vs reference" : "standard deep order vs reference");
            if (uns) CHECK(got.entries[0] == cdouble(0.0, 0.0), "unscaled: seed below the window never counts");
            else CHECK(got.entries[0] != cdouble(0.0, 0.0), "standard: the ladder activates the deep stream");
        }
        sht::ScaleLadder custom;
        custom.hi = 0x1p256;
        bool threw = false;
        try { (void)sht::compute_delta_a(alm, x, ms, custom); } catch (const std::invalid_argument&) { threw = true; }
        CHECK(threw, "non-reference ladder window rejected");
    }
    // argument errors (test_transforms.cpp:426-470)
    {
        auto [x, w] = sht::gauss_legendre_nodes(8);
        auto alm = make_random_alm(6, 6, 9);
        int n = 0;
        try { (void)sht::compute_delta_a(alm, x, std::vector<int>{1, 1}); } catch (const std::invalid_argument&) { ++n; }
        try { (void)sht::compute_delta_a(alm, x, std::vector<int>{-1}); } catch (const std::invalid_argument&) { ++n; }
        try { (void)sht::compute_delta_a(alm, x, std::vector<int>{0, 7}); } catch (const std::invalid_argument&) { ++n; }
        try { (void)sht::compute_delta_a(alm, std::vector<double>{1.5}, std::vector<int>{0}); } catch (const std::invalid_argument&) { ++n; }
        try { (void)sht::compute_delta_a_ring_major(alm, x, std::vector<int>{0}, 0); } catch (const std::invalid_argument&) { ++n; }
        sht::SkyMap bad;
        bad.grid = sht::build_healpix_grid(1);
        bad.pixels.assign(5, 0.0);
        try { (void)sht::analysis(bad, 4, 4); } catch (const std::invalid_argument&) { ++n; }
        sht::AlmSet tiny(2, 2);
        sht::PixelGrid empty;
        try { (void)sht::synthesis(tiny, empty); } catch (const std::invalid_argument&) { ++n; }
        CHECK(n == 7, "argument errors raise std::invalid_argument");
    }
    std::printf("PASS %d\n", passes);
    if (fails) std::printf("FAILURES %d\n", fails);
    return fails ? 1 : 0;
}
