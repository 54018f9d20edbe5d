// TEST INFRASTRUCTURE ONLY — the parity checker, never the product.
//
// C shim over the UNMODIFIED reference implementation (/root/reference/proj/src/*.cpp),
// compiled from the reference's own sources by oracle/build_ref.sh into
// oracle/_ref/libsht_ref.so with -Dsht=sht_ref.  Only tests/, bench.py's cpu_baseline /
// --impl reference leg and __graft_entry__.smoke() may load it.
//
// Every entry point forwards to the reference's public C++ API:
//   grid      -> build_healpix_grid / build_gauss_legendre_grid   (grid.hpp:45-58)
//   legendre  -> log_mu / beta_lm / plm_row / plm_row_scaled      (legendre.hpp:10-132)
//   inputs    -> splitmix64_at / uniform_pm1 / random_alm          (experiment.hpp:14-25)
//   transforms-> synthesis / analysis / compute_delta_a[_ring_major] / accumulate_alm
//                                                                   (transforms.hpp:32-79)
//   fourier   -> ring_synthesis_into / ring_analysis_into           (fourier.hpp:22-31)
//   distribution -> assign_m / assign_rings / distributed_synthesis / distributed_analysis
//                                                                   (distribution.hpp:15-77)
// Grids are passed as plain ring arrays so any PixelGrid can be reconstructed.
// Errors: every function returns 0 on success, 1 on std::invalid_argument,
// 2 on std::domain_error, 3 on any other exception; the message is kept for ref_last_error().

#include <cstdint>
#include <cmath>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "sht/distribution.hpp"
#include "sht/experiment.hpp"
#include "sht/fourier.hpp"
#include "sht/grid.hpp"
#include "sht/legendre.hpp"
#include "sht/perfmodel.hpp"
#include "sht/transforms.hpp"

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

sht::PixelGrid make_grid(int scheme, int nside, int n_rings, const double* cos_theta,
                         const int32_t* n_phi, const double* phi_0, const double* weight) {
    sht::PixelGrid g;
    g.scheme = scheme == 0 ? sht::GridScheme::healpix_ring : sht::GridScheme::gauss_legendre;
    g.nside = nside;
    g.rings.resize(static_cast<std::size_t>(n_rings));
    std::int64_t off = 0;
    for (int k = 0; k < n_rings; ++k) {
        sht::RingDescriptor& r = g.rings[static_cast<std::size_t>(k)];
        r.index = k;
        r.cos_theta = cos_theta[k];
        r.sin_theta = std::sqrt((1.0 - cos_theta[k]) * (1.0 + cos_theta[k]));
        r.n_phi = n_phi[k];
        r.phi_0 = phi_0[k];
        r.weight = weight[k];
        r.pixel_offset = off;
        off += n_phi[k];
    }
    g.n_pix = off;
    return g;
}

sht::AlmSet make_alm(int lmax, int mmax, const double* alm) {
    sht::AlmSet a(lmax, mmax);
    std::memcpy(a.values.data(), alm, a.values.size() * sizeof(sht::cdouble));
    return a;
}

sht::TransformOptions topts(int pairing, int kernel, std::uint64_t* steps) {
    sht::TransformOptions o;
    o.pairing = pairing ? sht::PairPolicy::mirror : sht::PairPolicy::none;
    o.kernel = kernel ? sht::KernelOrder::ring_major : sht::KernelOrder::m_major;
    o.step_counter = steps;
    return o;
}

void export_grid(const sht::PixelGrid& g, double* cos_theta, int32_t* n_phi, double* phi_0,
                 double* weight, int64_t* pixel_offset) {
    for (std::size_t k = 0; k < g.rings.size(); ++k) {
        const auto& r = g.rings[k];
        if (cos_theta) cos_theta[k] = r.cos_theta;
        if (n_phi) n_phi[k] = r.n_phi;
        if (phi_0) phi_0[k] = r.phi_0;
        if (weight) weight[k] = r.weight;
        if (pixel_offset) pixel_offset[k] = r.pixel_offset;
    }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- grid -------------------------------------------------------------------------------
int ref_healpix_grid(int nside, double* cos_theta, int32_t* n_phi, double* phi_0,
                     double* weight, int64_t* pixel_offset) {
    return guarded([&] {
        export_grid(sht::build_healpix_grid(nside), cos_theta, n_phi, phi_0, weight,
                    pixel_offset);
    });
}

int ref_gl_grid(int n_rings, int n_phi_each, double* cos_theta, int32_t* n_phi, double* phi_0,
                double* weight, int64_t* pixel_offset) {
    return guarded([&] {
        export_grid(sht::build_gauss_legendre_grid(n_rings, n_phi_each), cos_theta, n_phi,
                    phi_0, weight, pixel_offset);
    });
}

int ref_gl_nodes(int n, double* x, double* w) {
    return guarded([&] {
        auto [xs, ws] = sht::gauss_legendre_nodes(n);
        std::memcpy(x, xs.data(), xs.size() * sizeof(double));
        std::memcpy(w, ws.data(), ws.size() * sizeof(double));
    });
}

// ---- legendre ---------------------------------------------------------------------------
int ref_log_mu(int m, double* out) {
    return guarded([&] { *out = sht::log_mu(m); });
}
int ref_beta_lm(int l, int m, double* out) {
    return guarded([&] { *out = sht::beta_lm(l, m); });
}
int ref_pmm_from_log(int m, double x, double log_mu_m, double* mant, int32_t* scale) {
    return guarded([&] {
        auto v = sht::pmm_from_log(m, x, log_mu_m);
        *mant = v.mantissa;
        *scale = v.scale;
    });
}
int ref_plm_row(int m, double x, int lmax, int unscaled, double* out) {
    return guarded([&] {
        auto row = sht::plm_row(m, x, lmax,
                                unscaled ? sht::ScaleLadder::unscaled() : sht::ScaleLadder::standard());
        std::memcpy(out, row.data(), row.size() * sizeof(double));
    });
}
int ref_plm_row_scaled(int m, double x, int lmax, double* mant, int32_t* scale) {
    return guarded([&] {
        auto row = sht::plm_row_scaled(m, x, lmax);
        for (std::size_t i = 0; i < row.size(); ++i) {
            mant[i] = row[i].mantissa;
            scale[i] = row[i].scale;
        }
    });
}

// ---- inputs -----------------------------------------------------------------------------
uint64_t ref_splitmix64_at(uint64_t seed, uint64_t index) { return sht::splitmix64_at(seed, index); }
double ref_uniform_pm1(uint64_t seed, uint64_t index) { return sht::uniform_pm1(seed, index); }
int ref_random_alm(int lmax, int mmax, uint64_t seed, double* out) {
    return guarded([&] {
        auto a = sht::random_alm(lmax, mmax, seed);
        std::memcpy(out, a.values.data(), a.values.size() * sizeof(sht::cdouble));
    });
}

// ---- whole-sphere transforms (transforms.cpp:402-485) -----------------------------------
int ref_synthesis(int lmax, int mmax, const double* alm, int scheme, int nside, int n_rings,
                  const double* cos_theta, const int32_t* n_phi, const double* phi_0,
                  const double* weight, int pairing, int kernel, double* map_out,
                  uint64_t* steps) {
    return guarded([&] {
        auto grid = make_grid(scheme, nside, n_rings, cos_theta, n_phi, phi_0, weight);
        auto a = make_alm(lmax, mmax, alm);
        auto m = sht::synthesis(a, grid, topts(pairing, kernel, steps));
        std::memcpy(map_out, m.pixels.data(), m.pixels.size() * sizeof(double));
    });
}

int ref_analysis(int lmax, int mmax, const double* map, int scheme, int nside, int n_rings,
                 const double* cos_theta, const int32_t* n_phi, const double* phi_0,
                 const double* weight, int pairing, double* alm_out, uint64_t* steps) {
    return guarded([&] {
        sht::SkyMap sm;
        sm.grid = make_grid(scheme, nside, n_rings, cos_theta, n_phi, phi_0, weight);
        sm.pixels.assign(map, map + sm.grid.n_pix);
        auto a = sht::analysis(sm, lmax, mmax, topts(pairing, 0, steps));
        std::memcpy(alm_out, a.values.data(), a.values.size() * sizeof(sht::cdouble));
    });
}

// ---- Legendre-stage operators (transforms.cpp:269-365) ----------------------------------
int ref_compute_delta_a(int lmax, int mmax, const double* alm, int n_lat, const double* x,
                        int n_m, const int32_t* ms, int ring_major, int n_work_items,
                        int unscaled, double* delta_out, uint64_t* steps) {
    return guarded([&] {
        auto a = make_alm(lmax, mmax, alm);
        std::vector<double> lat(x, x + n_lat);
        std::vector<int> mset(ms, ms + n_m);
        const auto& ladder = unscaled ? sht::ScaleLadder::unscaled() : sht::ScaleLadder::standard();
        auto p = ring_major ? sht::compute_delta_a_ring_major(a, lat, mset, n_work_items, ladder, steps)
                            : sht::compute_delta_a(a, lat, mset, ladder, steps);
        std::memcpy(delta_out, p.entries.data(), p.entries.size() * sizeof(sht::cdouble));
    });
}

int ref_accumulate_alm(int lmax, int mmax, int n_lat, const double* x, int n_m,
                       const int32_t* ms, const double* delta, double* alm_out,
                       uint64_t* steps) {
    return guarded([&] {
        sht::DeltaPanel p;
        p.kind = sht::DeltaKind::analysis;
        p.rings.resize(static_cast<std::size_t>(n_lat));
        for (int i = 0; i < n_lat; ++i) p.rings[static_cast<std::size_t>(i)] = i;
        p.ms.assign(ms, ms + n_m);
        p.entries.resize(static_cast<std::size_t>(n_lat) * static_cast<std::size_t>(n_m));
        std::memcpy(p.entries.data(), delta, p.entries.size() * sizeof(sht::cdouble));
        std::vector<double> lat(x, x + n_lat);
        auto a = sht::accumulate_alm(p, lat, lmax, mmax, sht::ScaleLadder::standard(), steps);
        std::memcpy(alm_out, a.values.data(), a.values.size() * sizeof(sht::cdouble));
    });
}

// ---- per-ring Fourier stage (fourier.cpp:10-56) -----------------------------------------
int ref_ring_synthesis(int n_delta, const double* delta, int n_phi, double phi_0, double* out) {
    return guarded([&] {
        sht::RingDescriptor ring;
        ring.n_phi = n_phi;
        ring.phi_0 = phi_0;
        ring.weight = 1.0;
        std::vector<sht::cdouble> d(static_cast<std::size_t>(n_delta));
        std::memcpy(d.data(), delta, d.size() * sizeof(sht::cdouble));
        std::vector<double> o(static_cast<std::size_t>(n_phi > 0 ? n_phi : 0));
        sht::ring_synthesis_into(d, ring, o);
        std::memcpy(out, o.data(), o.size() * sizeof(double));
    });
}

int ref_ring_analysis(int n_phi, const double* samples, double phi_0, double weight, int mmax,
                      double* out) {
    return guarded([&] {
        sht::RingDescriptor ring;
        ring.n_phi = n_phi;
        ring.phi_0 = phi_0;
        ring.weight = weight;
        std::vector<double> s(samples, samples + n_phi);
        std::vector<sht::cdouble> o(static_cast<std::size_t>(mmax) + 1);
        sht::ring_analysis_into(s, ring, mmax, o);
        std::memcpy(out, o.data(), o.size() * sizeof(sht::cdouble));
    });
}

// ---- distribution (distribution.cpp:82-490) ---------------------------------------------
// Sets are returned flattened: counts[w] entries each, concatenated in worker order.
int ref_assign_m(int mmax, int n_workers, int32_t* counts, int32_t* flat) {
    return guarded([&] {
        auto s = sht::assign_m(mmax, n_workers);
        std::size_t k = 0;
        for (std::size_t w = 0; w < s.size(); ++w) {
            counts[w] = static_cast<int32_t>(s[w].size());
            for (int m : s[w]) flat[k++] = m;
        }
    });
}

int ref_assign_rings_healpix(int nside, int n_workers, int32_t* counts, int32_t* flat) {
    return guarded([&] {
        auto s = sht::assign_rings(sht::build_healpix_grid(nside), n_workers);
        std::size_t k = 0;
        for (std::size_t w = 0; w < s.size(); ++w) {
            counts[w] = static_cast<int32_t>(s[w].size());
            for (int r : s[w]) flat[k++] = r;
        }
    });
}

int ref_thread_partition(int n, const int32_t* ms, int n_threads, int32_t* counts,
                         int32_t* flat) {
    return guarded([&] {
        std::vector<int> v(ms, ms + n);
        auto s = sht::thread_partition(v, n_threads);
        std::size_t k = 0;
        for (std::size_t t = 0; t < s.size(); ++t) {
            counts[t] = static_cast<int32_t>(s[t].size());
            for (int m : s[t]) flat[k++] = m;
        }
    });
}

// stage_s[4] = precompute, recurrence, exchange, fft seconds; totals[2] = exchange bytes, steps
int ref_distributed_synthesis(int lmax, int mmax, const double* alm, int scheme, int nside,
                              int n_rings, const double* cos_theta, const int32_t* n_phi,
                              const double* phi_0, const double* weight, int n_workers,
                              int n_threads, int pairing, int kernel, double* map_out,
                              double* stage_s, uint64_t* totals) {
    return guarded([&] {
        auto grid = make_grid(scheme, nside, n_rings, cos_theta, n_phi, phi_0, weight);
        auto a = make_alm(lmax, mmax, alm);
        auto layout = sht::WorkerLayout::create(grid, mmax, n_workers);
        sht::Profiler prof;
        sht::RunOptions o;
        o.n_threads = n_threads;
        o.pairing = pairing ? sht::PairPolicy::mirror : sht::PairPolicy::none;
        o.kernel = kernel ? sht::KernelOrder::ring_major : sht::KernelOrder::m_major;
        o.profiler = &prof;
        auto m = sht::distributed_synthesis(a, grid, layout, o);
        std::memcpy(map_out, m.pixels.data(), m.pixels.size() * sizeof(double));
        if (stage_s) {
            stage_s[0] = prof.precompute_s;
            stage_s[1] = prof.recurrence_s;
            stage_s[2] = prof.exchange_s;
            stage_s[3] = prof.fft_s;
        }
        if (totals) {
            totals[0] = prof.exchange_bytes;
            totals[1] = prof.total_steps();
        }
    });
}

int ref_distributed_analysis(int lmax, int mmax, const double* map, int scheme, int nside,
                             int n_rings, const double* cos_theta, const int32_t* n_phi,
                             const double* phi_0, const double* weight, int n_workers,
                             int n_threads, int pairing, int kernel, double* alm_out,
                             double* stage_s, uint64_t* totals) {
    return guarded([&] {
        sht::SkyMap sm;
        sm.grid = make_grid(scheme, nside, n_rings, cos_theta, n_phi, phi_0, weight);
        sm.pixels.assign(map, map + sm.grid.n_pix);
        auto layout = sht::WorkerLayout::create(sm.grid, mmax, n_workers);
        sht::Profiler prof;
        sht::RunOptions o;
        o.n_threads = n_threads;
        o.pairing = pairing ? sht::PairPolicy::mirror : sht::PairPolicy::none;
        o.kernel = kernel ? sht::KernelOrder::ring_major : sht::KernelOrder::m_major;
        o.profiler = &prof;
        auto a = sht::distributed_analysis(sm, lmax, mmax, layout, o);
        std::memcpy(alm_out, a.values.data(), a.values.size() * sizeof(sht::cdouble));
        if (stage_s) {
            stage_s[0] = prof.precompute_s;
            stage_s[1] = prof.recurrence_s;
            stage_s[2] = prof.exchange_s;
            stage_s[3] = prof.fft_s;
        }
        if (totals) {
            totals[0] = prof.exchange_bytes;
            totals[1] = prof.total_steps();
        }
    });
}

}  // extern "C"
