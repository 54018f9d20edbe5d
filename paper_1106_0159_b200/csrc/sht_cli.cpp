// sht_b200: the reference CLI's subcommands (tools/sht_main.cpp:98-277) on the GPU path.
//   sht_b200 grid info    [--grid healpix|gauss-legendre] [--nside N] [--nrings R] [--nphi P]
//   sht_b200 synth  [input.alm] --out map.shtmap [--lmax L] [--mmax M] [--seed S] [--workers W]
//   sht_b200 analyze input.shtmap --out out.alm [--lmax L] [--mmax M] [--workers W]
//   sht_b200 roundtrip [--out back.alm] ...        prints D_err
//   sht_b200 bench [--csv report.csv] ...          profiled synthesis + cost report (B200 model)
//   sht_b200 model [--nside N ...] [--workers W ...] [--b200] [--csv out.csv]
//   sht_b200 partition ...                         worker / thread decomposition
// Argument errors and library exceptions exit with status 1 ("error: ..."), as the reference.
#include <cstdint>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "sht/distribution.hpp"
#include "sht/experiment.hpp"
#include "sht/io.hpp"
#include "sht/perfmodel.hpp"

namespace {

struct Cfg {
    std::string grid = "healpix";
    int nside = 64, nrings = 0, nphi = 0, lmax = 128, mmax = -1;
    std::uint64_t seed = 12345;
    int workers = 1, threads = 1;
    std::string kernel = "m-major", out, csv, input;
    std::vector<int> sweep_nside, sweep_workers;
    bool b200 = false;
};

int to_int(const std::string& v, const std::string& k) {
    try {
        size_t pos = 0;
        const long x = std::stol(v, &pos);
        if (pos != v.size()) throw std::invalid_argument(k);
        return static_cast<int>(x);
    } catch (const std::exception&) {
        throw std::invalid_argument("bad value for " + k + ": " + v);
    }
}

Cfg parse(int argc, char** argv, int first) {
    Cfg c;
    if (const char* t = std::getenv("SHT_THREADS")) c.threads = to_int(t, "SHT_THREADS");
    for (int i = first; i < argc; ++i) {
        const std::string a = argv[i];
        auto val = [&]() -> std::string {
            if (i + 1 >= argc) throw std::invalid_argument(a + " needs a value");
            return argv[++i];
        };
        if (a == "--grid") c.grid = val();
        else if (a == "--nside") { c.nside = to_int(val(), a); c.sweep_nside.push_back(c.nside); }
        else if (a == "--nrings") c.nrings = to_int(val(), a);
        else if (a == "--nphi") c.nphi = to_int(val(), a);
        else if (a == "--lmax") c.lmax = to_int(val(), a);
        else if (a == "--mmax") c.mmax = to_int(val(), a);
        else if (a == "--seed") c.seed = std::stoull(val());
        else if (a == "--workers") { c.workers = to_int(val(), a); c.sweep_workers.push_back(c.workers); }
        else if (a == "--threads") c.threads = to_int(val(), a);
        else if (a == "--kernel") c.kernel = val();
        else if (a == "--out") c.out = val();
        else if (a == "--csv") c.csv = val();
        else if (a == "--b200") c.b200 = true;
        else if (!a.empty() && a[0] != '-' && c.input.empty()) c.input = a;
        else throw std::invalid_argument("unknown argument " + a);
    }
    if (c.grid != "healpix" && c.grid != "gauss-legendre") throw std::invalid_argument("--grid: healpix or gauss-legendre");
    if (c.kernel != "m-major" && c.kernel != "ring-major") throw std::invalid_argument("--kernel: m-major or ring-major");
    return c;
}

sht::PixelGrid make_grid(const Cfg& c) {
    if (c.grid == "healpix") return sht::build_healpix_grid(c.nside);
    const int nr = c.nrings > 0 ? c.nrings : c.lmax + 1;
    return sht::build_gauss_legendre_grid(nr, c.nphi > 0 ? c.nphi : 2 * nr);
}

int mmax_of(const Cfg& c) { return c.mmax >= 0 ? c.mmax : c.lmax; }

sht::RunOptions opts(const Cfg& c, sht::Profiler* p = nullptr) {
    sht::RunOptions o;
    o.n_threads = c.threads;
    o.kernel = c.kernel == "ring-major" ? sht::KernelOrder::ring_major : sht::KernelOrder::m_major;
    o.profiler = p;
    return o;
}

std::string join(const std::vector<int>& v) {
    std::ostringstream os;
    for (size_t i = 0; i < v.size(); ++i) os << (i ? " " : "") << v[i];
    return os.str();
}

int run(int argc, char** argv) {
    if (argc < 2) throw std::invalid_argument("usage: sht_b200 <grid|synth|analyze|roundtrip|bench|model|partition> ...");
    const std::string cmd = argv[1];
    if (cmd == "grid") {
        if (argc < 3 || std::string(argv[2]) != "info") throw std::invalid_argument("usage: sht_b200 grid info ...");
        const Cfg c = parse(argc, argv, 3);
        const auto g = make_grid(c);
        double w = 0.0;
        for (const auto& r : g.rings) w += r.weight * r.n_phi;
        std::cout << "scheme " << sht::to_string(g.scheme) << "\n";
        if (g.scheme == sht::GridScheme::healpix_ring) std::cout << "nside " << g.nside << "\n";
        std::cout << "rings " << g.n_rings() << "\npixels " << g.n_pix << "\n";
        std::cout.precision(15);
        std::cout << "weight_sum_over_4pi " << w / (4.0 * 3.14159265358979323846) << "\n";
        return 0;
    }
    const Cfg c = parse(argc, argv, 2);
    if (cmd == "synth") {
        const auto g = make_grid(c);
        const auto alm = c.input.empty() ? sht::random_alm(c.lmax, mmax_of(c), c.seed) : sht::read_alm(c.input);
        const auto map = sht::distributed_synthesis(alm, g, sht::WorkerLayout::create(g, alm.mmax, c.workers), opts(c));
        if (c.out.empty()) throw std::runtime_error("synth: --out is required");
        sht::write_map(c.out, map);
        std::cout << "wrote " << c.out << " (" << map.pixels.size() << " pixels)\n";
    } else if (cmd == "analyze") {
        if (c.input.empty()) throw std::invalid_argument("analyze: input map required");
        const auto map = sht::read_map(c.input);
        const auto alm = sht::distributed_analysis(map, c.lmax, mmax_of(c),
                                                   sht::WorkerLayout::create(map.grid, mmax_of(c), c.workers), opts(c));
        if (c.out.empty()) throw std::runtime_error("analyze: --out is required");
        sht::write_alm(c.out, alm);
        std::cout << "wrote " << c.out << " (" << alm.values.size() << " coefficients)\n";
    } else if (cmd == "roundtrip") {
        const auto g = make_grid(c);
        const auto alm = sht::random_alm(c.lmax, mmax_of(c), c.seed);
        const auto lay = sht::WorkerLayout::create(g, mmax_of(c), c.workers);
        const auto map = sht::distributed_synthesis(alm, g, lay, opts(c));
        const auto back = sht::distributed_analysis(map, c.lmax, mmax_of(c), lay, opts(c));
        std::cout.precision(17);
        std::cout << "D_err " << sht::roundtrip_error(alm, back) << "\n";
        if (!c.out.empty()) sht::write_alm(c.out, back);
    } else if (cmd == "bench") {
        const auto g = make_grid(c);
        const auto alm = sht::random_alm(c.lmax, mmax_of(c), c.seed);
        sht::Profiler prof;
        // first call plans (tables, activation scan, ring FFT tables); the profiled one runs warm
        (void)sht::distributed_synthesis(alm, g, sht::WorkerLayout::create(g, mmax_of(c), c.workers), opts(c));
        const auto map = sht::distributed_synthesis(alm, g, sht::WorkerLayout::create(g, mmax_of(c), c.workers), opts(c, &prof));
        if (!c.out.empty()) sht::write_map(c.out, map);
        const auto rep = sht::build_report(g.n_rings(), c.lmax, mmax_of(c), c.workers, &prof, sht::CostParams::b200());
        if (!c.csv.empty()) {
            std::ofstream os(c.csv, std::ios::trunc);
            if (!os) throw std::runtime_error("bench: cannot open " + c.csv);
            rep.write_csv(os);
        } else {
            rep.write_csv(std::cout);
        }
        std::cout.precision(6);
        std::cout << "recurrence_steps " << prof.total_steps() << "\nrecurrence_s " << prof.recurrence_s
                  << "\nfft_s " << prof.fft_s << "\n";
    } else if (cmd == "model") {
        const std::vector<int> ns = c.sweep_nside.empty() ? std::vector<int>{256, 512, 1024} : c.sweep_nside;
        const std::vector<int> ws = c.sweep_workers.empty() ? std::vector<int>{1, 2, 4, 8, 16} : c.sweep_workers;
        const auto p = c.b200 ? sht::CostParams::b200() : sht::CostParams{};
        if (!c.csv.empty()) {
            std::ofstream os(c.csv, std::ios::trunc);
            if (!os) throw std::runtime_error("model: cannot open " + c.csv);
            sht::runtime_curves(os, ns, ws, p);
        } else {
            sht::runtime_curves(std::cout, ns, ws, p);
        }
    } else if (cmd == "partition") {
        const auto g = make_grid(c);
        const auto lay = sht::WorkerLayout::create(g, mmax_of(c), c.workers);
        auto steps = [&](const std::vector<int>& ms) {
            std::uint64_t s = 0;
            for (int m : ms) s += static_cast<std::uint64_t>(c.lmax - m + 1);
            return s * static_cast<std::uint64_t>(g.n_rings());
        };
        for (int w = 0; w < lay.n_workers; ++w) {
            std::cout << "worker " << w << " m { " << join(lay.m_sets[w]) << " }\n";
            std::cout << "worker " << w << " rings { " << join(lay.ring_sets[w]) << " }\n";
            std::cout << "worker " << w << " steps " << steps(lay.m_sets[w]) << "\n";
            const auto tp = sht::thread_partition(lay.m_sets[w], c.threads);
            for (int t = 0; t < c.threads; ++t)
                std::cout << "worker " << w << " thread " << t << " m { " << join(tp[t]) << " } steps " << steps(tp[t]) << "\n";
        }
    } else {
        throw std::invalid_argument("unknown subcommand " + cmd);
    }
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        return run(argc, argv);
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
