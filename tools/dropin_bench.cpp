// The reference C++ API as a reference user calls it (sht::synthesis / sht::analysis on
// std::vector-backed AlmSet / SkyMap) at C4 through libsht_b200.so: wall-clock ms per call,
// median of 5 after a warm-up, and the part spent allocating and zero-filling the returned
// containers.
//
//   g++ -std=c++20 -O2 -I include tools/dropin_bench.cpp -L paper_1106_0159_b200 -lsht_b200 -lshtc \
//       -Wl,-rpath,$PWD/paper_1106_0159_b200 -o tools/dropin_bench.bin
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <random>
#include <vector>

#include "sht/alm.hpp"
#include "sht/grid.hpp"
#include "sht/transforms.hpp"

static double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main(int argc, char** argv) {
    const int nside = argc > 1 ? std::atoi(argv[1]) : 2048, lmax = 2 * nside;
    const sht::PixelGrid grid = sht::build_healpix_grid(nside);
    sht::AlmSet alm(lmax, lmax);
    std::mt19937_64 rng(12345);
    std::normal_distribution<double> nd;
    for (auto& v : alm.values) v = {nd(rng), nd(rng)};
    sht::TransformOptions o;
    o.pairing = sht::PairPolicy::mirror;
    sht::SkyMap m = sht::synthesis(alm, grid, o);  // warm-up (plans)
    sht::AlmSet b = sht::analysis(m, lmax, lmax, o);
    std::vector<double> ts, ta, tz;
    for (int r = 0; r < 5; ++r) {
        const double t0 = now_ms();
        sht::SkyMap m2 = sht::synthesis(alm, grid, o);
        const double t1 = now_ms();
        sht::AlmSet b2 = sht::analysis(m2, lmax, lmax, o);
        const double t2 = now_ms();
        std::vector<double> z(static_cast<size_t>(grid.n_pix), 0.0);  // the SkyMap's own zero fill
        const double t3 = now_ms();
        ts.push_back(t1 - t0);
        ta.push_back(t2 - t1);
        tz.push_back(t3 - t2);
    }
    auto med = [](std::vector<double> v) { std::sort(v.begin(), v.end()); return v[v.size() / 2]; };
    std::printf("drop-in nside %d lmax %d: synthesis %.2f ms, analysis %.2f ms; a %.0f MB zero-filled vector alone %.2f ms\n",
                nside, lmax, med(ts), med(ta), grid.n_pix * 8 / 1e6, med(tz));
    return 0;
}
