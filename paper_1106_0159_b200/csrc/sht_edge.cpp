// Edge of the drop-in: SHTMAP1/SHTALM1 containers and the
// alpha-beta-gamma performance model with B200 recalibration.  Host code; same formats and
// formulas as the reference (src/io.cpp:98-167, src/perfmodel.cpp:9-119).
#include <algorithm>
#include <bit>
#include <cmath>
#include <cstdint>
#include <fstream>
#include <ostream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "sht/io.hpp"
#include "sht/perfmodel.hpp"

namespace sht {

namespace {

using Header = std::vector<std::pair<std::string, std::string>>;

void put_f64(std::ostream& os, const double* d, size_t n) {
    if constexpr (std::endian::native == std::endian::little) {
        os.write(reinterpret_cast<const char*>(d), static_cast<std::streamsize>(n * 8));
    } else {
        for (size_t i = 0; i < n; ++i) {
            const uint64_t u = __builtin_bswap64(std::bit_cast<uint64_t>(d[i]));
            os.write(reinterpret_cast<const char*>(&u), 8);
        }
    }
}

void get_f64(std::istream& is, double* d, size_t n, const char* what) {
    is.read(reinterpret_cast<char*>(d), static_cast<std::streamsize>(n * 8));
    if (static_cast<size_t>(is.gcount()) != n * 8) throw std::runtime_error(std::string(what) + ": truncated payload");
    if constexpr (std::endian::native != std::endian::little)
        for (size_t i = 0; i < n; ++i) d[i] = std::bit_cast<double>(__builtin_bswap64(std::bit_cast<uint64_t>(d[i])));
}

Header header(std::istream& is, const char* magic, const char* what) {
    std::string line;
    if (!std::getline(is, line) || line != magic) throw std::runtime_error(std::string(what) + ": not a " + magic + " file");
    Header h;
    while (std::getline(is, line)) {
        if (line == "end") return h;
        const auto sp = line.find(' ');
        if (sp == std::string::npos || sp == 0 || sp + 1 >= line.size())
            throw std::runtime_error(std::string(what) + ": malformed header line '" + line + "'");
        h.emplace_back(line.substr(0, sp), line.substr(sp + 1));
    }
    throw std::runtime_error(std::string(what) + ": header missing 'end'");
}

const std::string& field(const Header& h, const std::string& key, const char* what) {
    for (const auto& [k, v] : h)
        if (k == key) return v;
    throw std::runtime_error(std::string(what) + ": missing header field " + key);
}

long long ifield(const Header& h, const std::string& key, const char* what) {
    try {
        return std::stoll(field(h, key, what));
    } catch (const std::invalid_argument&) {
        throw std::runtime_error(std::string(what) + ": bad value for " + key);
    } catch (const std::out_of_range&) {
        throw std::runtime_error(std::string(what) + ": bad value for " + key);
    }
}

}  // namespace

void write_map(const std::string& path, const SkyMap& map) {
    if (map.pixels.size() != static_cast<size_t>(map.grid.n_pix))
        throw std::invalid_argument("write_map: pixel count != grid");
    std::ofstream os(path, std::ios::binary | std::ios::trunc);
    if (!os) throw std::runtime_error("write_map: cannot open " + path);
    std::ostringstream h;
    h << "SHTMAP1\n";
    if (map.grid.scheme == GridScheme::healpix_ring) {
        h << "scheme healpix-ring\nnside " << map.grid.nside << "\n";
    } else {
        h << "scheme gauss-legendre\nnrings " << map.grid.n_rings() << "\nnphi "
          << (map.grid.n_rings() ? map.grid.rings[0].n_phi : 0) << "\n";
    }
    h << "npix " << map.grid.n_pix << "\nend\n";
    os << h.str();
    put_f64(os, map.pixels.data(), map.pixels.size());
    if (!os) throw std::runtime_error("write_map: write failed for " + path);
}

SkyMap read_map(const std::string& path) {
    std::ifstream is(path, std::ios::binary);
    if (!is) throw std::runtime_error("read_map: cannot open " + path);
    const Header h = header(is, "SHTMAP1", "read_map");
    const std::string scheme = field(h, "scheme", "read_map");
    SkyMap map;
    if (scheme == "healpix-ring")
        map.grid = build_healpix_grid(static_cast<int>(ifield(h, "nside", "read_map")));
    else if (scheme == "gauss-legendre")
        map.grid = build_gauss_legendre_grid(static_cast<int>(ifield(h, "nrings", "read_map")),
                                             static_cast<int>(ifield(h, "nphi", "read_map")));
    else
        throw std::runtime_error("read_map: unknown scheme " + scheme);
    if (ifield(h, "npix", "read_map") != map.grid.n_pix)
        throw std::runtime_error("read_map: npix inconsistent with grid parameters");
    map.pixels.resize(static_cast<size_t>(map.grid.n_pix));
    get_f64(is, map.pixels.data(), map.pixels.size(), "read_map");
    return map;
}

void write_alm(const std::string& path, const AlmSet& alm) {
    std::ofstream os(path, std::ios::binary | std::ios::trunc);
    if (!os) throw std::runtime_error("write_alm: cannot open " + path);
    os << "SHTALM1\nlmax " << alm.lmax << "\nmmax " << alm.mmax << "\nend\n";
    put_f64(os, reinterpret_cast<const double*>(alm.values.data()), alm.values.size() * 2);
    if (!os) throw std::runtime_error("write_alm: write failed for " + path);
}

AlmSet read_alm(const std::string& path) {
    std::ifstream is(path, std::ios::binary);
    if (!is) throw std::runtime_error("read_alm: cannot open " + path);
    const Header h = header(is, "SHTALM1", "read_alm");
    const int lmax = static_cast<int>(ifield(h, "lmax", "read_alm"));
    const int mmax = static_cast<int>(ifield(h, "mmax", "read_alm"));
    if (lmax < 0 || mmax < 0 || lmax < mmax) throw std::runtime_error("read_alm: bad band limits");
    AlmSet a(lmax, mmax);
    get_f64(is, reinterpret_cast<double*>(a.values.data()), a.values.size() * 2, "read_alm");
    return a;
}

// ---- performance model ----------------------------------------------------------------------
CostParams CostParams::b200() {
    CostParams p;
    p.alpha = 1.1e-5;            // one fused-exchange barrier round per worker, launch included:
                                 // 22.8 us for 2 workers, 75.7 us for 8 on one B200
                                 // (tools/calibrate_exchange.py, profiles/r02_exchange_calibration.json)
    p.beta_inv_bw = 1.0 / 770e9; // peer copy per direction per GPU as the B200 profiling guide
                                 // measured it (a 1-GPU box has no NVLink to time; fit_exchange
                                 // refits alpha and beta from multi-GPU samples)
    p.gamma = 1.42e-14;          // Legendre seconds per model flop at C4: (6.90 + 8.65) / 2 ms over
                                 // 4 R_N lmax mmax = 549.7 G (round 1, 1 GPU, profiles/r01_bench.json)
    return p;
}

FlopsBreakdown flops_estimate(double r_n, double lmax, double mmax, int n_workers) {
    if (n_workers < 1) throw std::invalid_argument("flops_estimate: n_workers must be >= 1");
    if (r_n < 0 || lmax < 0 || mmax < 0) throw std::invalid_argument("flops_estimate: negative problem size");
    FlopsBreakdown f;
    f.precompute = flops_c1 * mmax;
    f.recurrence = flops_c2 * r_n * lmax * mmax / n_workers;
    f.fft = flops_c3 * (r_n / n_workers) * mmax * std::log2(std::max(mmax, 2.0));
    return f;
}

double message_size(double r_n, double mmax, int n_workers, int n_c) {
    if (n_workers < 1) throw std::invalid_argument("message_size: n_workers must be >= 1");
    if (r_n < 0 || mmax < 0 || n_c < 1) throw std::invalid_argument("message_size: negative problem size");
    return r_n * (mmax / n_workers) * n_c;
}

double comm_time(double s, int n_workers, const CostParams& p) {
    if (n_workers < 1) throw std::invalid_argument("comm_time: n_workers must be >= 1");
    if (s < 0) throw std::invalid_argument("comm_time: negative message size");
    if (n_workers == 1) return 0.0;
    const double n = n_workers;
    if (s <= p.switch_bytes) return p.alpha * std::log2(n) + p.beta_inv_bw * s * (n / 2.0) * std::log2(n);
    return p.alpha * (n - 1.0) + p.beta_inv_bw * s * (n - 1.0);
}

void runtime_curves(std::ostream& os, std::span<const int> nsides, std::span<const int> workers,
                    const CostParams& p) {
    os << "nside,lmax,mmax,n_workers,precompute_s,compute_s,comm_s,ratio\n";
    os.precision(12);
    for (int ns : nsides) {
        if (ns < 1) throw std::invalid_argument("runtime_curves: nside must be >= 1");
        const double l = 2.0 * ns, r = 4.0 * ns - 1.0;
        for (int n : workers) {
            const auto f = flops_estimate(r, l, l, n);
            const double pre = p.gamma * f.precompute, comp = p.gamma * (f.recurrence + f.fft);
            const double comm = comm_time(message_size(r, l, n, p.n_c), n, p);
            os << ns << ',' << l << ',' << l << ',' << n << ',' << pre << ',' << comp << ',' << comm << ','
               << (comm > 0.0 ? comp / comm : 0.0) << '\n';
        }
    }
}

void CostReport::write_csv(std::ostream& os) const {
    os << "stage,predicted_s,measured_s,flops,bytes\n";
    os.precision(12);
    for (const auto& s : stages) {
        os << s.stage << ',' << s.predicted_s << ',';
        if (s.has_measured) os << s.measured_s;
        os << ',' << s.flops << ',' << s.bytes << '\n';
    }
}

CostReport build_report(double r_n, double lmax, double mmax, int n_workers, const Profiler* prof,
                        const CostParams& p) {
    const auto f = flops_estimate(r_n, lmax, mmax, n_workers);
    const double s = message_size(r_n, mmax, n_workers, p.n_c);
    CostReport rep;
    rep.stages = {{"precompute", p.gamma * f.precompute, false, 0.0, f.precompute, 0.0},
                  {"recurrence", p.gamma * f.recurrence, false, 0.0, f.recurrence, 0.0},
                  {"exchange", comm_time(s, n_workers, p), false, 0.0, 0.0,
                   s * n_workers * std::max(n_workers - 1, 0)},
                  {"fft", p.gamma * f.fft, false, 0.0, f.fft, 0.0}};
    if (prof) {
        const double m[4] = {prof->precompute_s, prof->recurrence_s, prof->exchange_s, prof->fft_s};
        for (int i = 0; i < 4; ++i) {
            rep.stages[i].has_measured = true;
            rep.stages[i].measured_s = m[i];
        }
        rep.stages[2].bytes = static_cast<double>(prof->exchange_bytes);
    }
    return rep;
}

namespace {
// comm_time = alpha * ca + beta * cb for the branch the message size selects
std::pair<double, double> comm_coeffs(double s, int n_workers, const CostParams& p) {
    if (n_workers <= 1) return {0.0, 0.0};
    const double n = n_workers;
    if (s <= p.switch_bytes) return {std::log2(n), s * (n / 2.0) * std::log2(n)};
    return {n - 1.0, s * (n - 1.0)};
}
}  // namespace

CostParams calibrate(const CostParams& base, double r_n, double lmax, double mmax, int n_workers,
                     const Profiler& prof) {
    CostParams p = base;
    const auto f = flops_estimate(r_n, lmax, mmax, n_workers);
    if (f.recurrence > 0 && prof.recurrence_s > 0) p.gamma = prof.recurrence_s / f.recurrence;
    if (n_workers > 1 && prof.exchange_s > 0 && prof.exchange_bytes > 0) {
        const auto [ca, cb] = comm_coeffs(message_size(r_n, mmax, n_workers, p.n_c), n_workers, p);
        const double rest = prof.exchange_s - p.alpha * ca;
        if (cb > 0 && rest > 0) p.beta_inv_bw = rest / cb;
    }
    return p;
}

CostParams fit_exchange(const CostParams& base, std::span<const ExchangeSample> samples) {
    // normal equations of min sum (alpha ca_i + beta cb_i - t_i)^2
    double aa = 0, ab = 0, bb = 0, at = 0, bt = 0;
    for (const auto& x : samples) {
        if (x.n_workers < 2 || x.msg_bytes < 0 || x.seconds < 0)
            throw std::invalid_argument("fit_exchange: samples need n_workers >= 2 and non-negative sizes");
        const auto [ca, cb] = comm_coeffs(x.msg_bytes, x.n_workers, base);
        aa += ca * ca;
        ab += ca * cb;
        bb += cb * cb;
        at += ca * x.seconds;
        bt += cb * x.seconds;
    }
    const double det = aa * bb - ab * ab;
    if (!(std::fabs(det) > 1e-12 * std::max(aa * bb, 1e-300)))
        throw std::invalid_argument("fit_exchange: samples do not determine alpha and beta");
    CostParams p = base;
    p.alpha = (at * bb - ab * bt) / det;
    p.beta_inv_bw = (aa * bt - ab * at) / det;
    return p;
}

}  // namespace sht
