// CPU checks of the drop-in edge (no GPU needed): perfmodel known answers
// (test_perfmodel.cpp:70-124) and SHTMAP1/SHTALM1 round trips (test_experiment.cpp:152-241).
#include <cmath>
#include <cstdio>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "sht/experiment.hpp"
#include "sht/grid.hpp"
#include "sht/io.hpp"
#include "sht/perfmodel.hpp"

static int fails = 0, passes = 0;
#define CHECK(c, w) do { if (c) ++passes; else { ++fails; std::printf("FAIL %s (line %d)\n", w, __LINE__); } } while (0)

template <class E, class F>
static bool throws(F f) {
    try { f(); } catch (const E&) { return true; } catch (...) { return false; }
    return false;
}

int main(int argc, char** argv) {
    const std::string dir = argc > 1 ? argv[1] : "/tmp";
    const auto fb = sht::flops_estimate(15, 8, 8, 1);
    CHECK(fb.recurrence == sht::flops_c2 * 960.0, "recurrence flops");
    CHECK(fb.precompute == sht::flops_c1 * 8.0, "precompute flops");
    CHECK(fb.fft == sht::flops_c3 * 15.0 * 8.0 * 3.0, "fft flops");
    CHECK(sht::flops_estimate(15, 8, 8, 2).recurrence == 0.5 * fb.recurrence, "split recurrence");
    CHECK(throws<std::invalid_argument>([] { sht::flops_estimate(15, 8, 8, 0); }), "flops n=0");
    CHECK(sht::message_size(15, 8, 4, 16) == 480.0, "message size");
    CHECK(sht::message_size(16383, 8192, 128, 16) == 16776192.0, "message size large");
    sht::CostParams p;
    CHECK(sht::comm_time(480, 1) == 0.0, "comm one worker");
    CHECK(std::fabs(sht::comm_time(480, 4, p) - 2.192e-5) < 1e-17, "short branch");
    CHECK(std::fabs(sht::comm_time(1048576, 4, p) - 3.175728e-3) < 1e-15, "long branch");
    CHECK(sht::comm_time(262144, 4, p) == p.alpha * 2.0 + p.beta_inv_bw * 262144.0 * 2.0 * 2.0, "switch inclusive");
    CHECK(throws<std::invalid_argument>([] { sht::comm_time(-1.0, 2); }), "negative message");
    std::ostringstream os;
    sht::runtime_curves(os, std::vector<int>{64}, std::vector<int>{1, 2}, p);
    CHECK(os.str().rfind("nside,lmax,mmax,n_workers,precompute_s,compute_s,comm_s,ratio\n", 0) == 0, "curves header");
    sht::Profiler prof;
    prof.configure(2, 1);
    prof.recurrence_s = 0.01;
    const auto cal = sht::calibrate(p, 255, 128, 128, 2, prof);
    CHECK(std::fabs(cal.gamma - 0.01 / sht::flops_estimate(255, 128, 128, 2).recurrence) < 1e-25, "calibrate gamma");
    // exchange recalibration: beta from a profiled exchange (alpha's share removed), and the
    // least-squares fit recovering known alpha / beta exactly from samples of both branches
    prof.exchange_s = 1e-3;
    prof.exchange_bytes = 123456;
    const double s_msg = sht::message_size(255, 128, 2, p.n_c);
    const auto cal2 = sht::calibrate(p, 255, 128, 128, 2, prof);
    CHECK(std::fabs(sht::comm_time(s_msg, 2, cal2) - 1e-3) < 1e-15, "calibrate beta reproduces the exchange");
    sht::CostParams truth;
    truth.alpha = 7.5e-6;
    truth.beta_inv_bw = 1.0 / 640e9;
    std::vector<sht::ExchangeSample> xs;
    for (int n : {2, 4, 8})
        for (double b : {4096.0, 1e5, 1e6, 3e7}) xs.push_back({n, b, sht::comm_time(b, n, truth)});
    const auto fit = sht::fit_exchange(p, xs);
    CHECK(std::fabs(fit.alpha - truth.alpha) < 1e-12 && std::fabs(fit.beta_inv_bw / truth.beta_inv_bw - 1.0) < 1e-9,
          "fit_exchange recovers alpha and beta");
    CHECK(throws<std::invalid_argument>([&] { sht::fit_exchange(p, std::span(xs.data(), 1)); }), "fit needs 2 samples");
    prof.exchange_s = 0.0;
    prof.exchange_bytes = 0;
    const auto rep = sht::build_report(255, 128, 128, 2, &prof, sht::CostParams::b200());
    CHECK(rep.stages.size() == 4 && rep.stages[1].has_measured && rep.stages[1].measured_s == 0.01, "report");
    // containers round trip bit for bit
    sht::SkyMap m;
    m.grid = sht::build_healpix_grid(4);
    m.pixels.resize(m.grid.n_pix);
    for (size_t i = 0; i < m.pixels.size(); ++i) m.pixels[i] = sht::uniform_pm1(7, i);
    sht::write_map(dir + "/t.shtmap", m);
    const auto m2 = sht::read_map(dir + "/t.shtmap");
    CHECK(m2.pixels == m.pixels && m2.grid.n_pix == m.grid.n_pix && m2.grid.nside == 4, "map round trip");
    sht::SkyMap g;
    g.grid = sht::build_gauss_legendre_grid(6, 13);
    g.pixels.assign(g.grid.n_pix, 0.25);
    sht::write_map(dir + "/g.shtmap", g);
    CHECK(sht::read_map(dir + "/g.shtmap").grid.n_pix == 78, "GL map round trip");
    const auto a = sht::random_alm(9, 7, 3);
    sht::write_alm(dir + "/t.shtalm", a);
    const auto a2 = sht::read_alm(dir + "/t.shtalm");
    CHECK(a2.values == a.values && a2.lmax == 9 && a2.mmax == 7, "alm round trip");
    { std::ofstream bad(dir + "/bad.shtalm"); bad << "SHTALM1\nlmax 3\nmmax 3\nend\nxx"; }
    CHECK(throws<std::runtime_error>([&] { sht::read_alm(dir + "/bad.shtalm"); }), "truncated payload");
    { std::ofstream bad(dir + "/bad2.shtmap"); bad << "SHTXXX1\n"; }
    CHECK(throws<std::runtime_error>([&] { sht::read_map(dir + "/bad2.shtmap"); }), "wrong magic");
    CHECK(throws<std::runtime_error>([&] { sht::read_map(dir + "/missing"); }), "missing file");
    std::printf("PASS %d\n", passes);
    return fails ? 1 : 0;
}
