// Drop-in geometry API (B200 build).  Same names, fields and semantics as the reference's
// include/sht/grid.hpp:13-66; implemented on the host in sht_dropin.cpp.
#pragma once

#include <cstdint>
#include <optional>
#include <string>
#include <utility>
#include <vector>

namespace sht {

// One iso-latitude ring; samples at phi_0 + j * 2*pi/n_phi.
struct RingDescriptor {
    int index = 0;
    double cos_theta = 0.0;
    double sin_theta = 0.0;
    int n_phi = 0;
    double phi_0 = 0.0;
    double weight = 0.0;
    std::int64_t pixel_offset = 0;
};

enum class GridScheme { healpix_ring, gauss_legendre };

struct PixelGrid {
    GridScheme scheme = GridScheme::healpix_ring;
    std::int64_t n_pix = 0;
    int nside = 0;
    std::vector<RingDescriptor> rings;

    int n_rings() const { return static_cast<int>(rings.size()); }
    std::vector<double> cos_thetas() const;
};

PixelGrid build_healpix_grid(int nside);
PixelGrid build_gauss_legendre_grid(int n_rings, int n_phi);
std::pair<std::vector<double>, std::vector<double>> gauss_legendre_nodes(int n);
std::vector<std::pair<int, std::optional<int>>> symmetric_ring_pairs(const PixelGrid& grid);
std::string to_string(GridScheme scheme);

}  // namespace sht
