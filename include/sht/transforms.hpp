// Drop-in transforms API (B200 build): alm2map / map2alm and the Legendre-stage operators
// with the reference's signatures (include/sht/transforms.hpp:16-79).  Every call runs on
// the GPU through the C ABI (include/shtc.h); there is no CPU path.
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "sht/alm.hpp"
#include "sht/legendre.hpp"

namespace sht {

enum class KernelOrder { m_major, ring_major };
enum class PairPolicy { none, mirror };

struct TransformOptions {
    KernelOrder kernel = KernelOrder::m_major;
    PairPolicy pairing = PairPolicy::none;
    std::uint64_t* step_counter = nullptr;  // += lmax-m+1 per (order, stream), nominal
};

DeltaPanel compute_delta_a(const AlmSet& alm, std::span<const double> cos_thetas,
                           std::span<const int> m_set,
                           const ScaleLadder& ladder = ScaleLadder::standard(),
                           std::uint64_t* step_counter = nullptr);

DeltaPanel compute_delta_a_ring_major(const AlmSet& alm, std::span<const double> cos_thetas,
                                      std::span<const int> m_set, int n_work_items = 1,
                                      const ScaleLadder& ladder = ScaleLadder::standard(),
                                      std::uint64_t* step_counter = nullptr);

AlmSet accumulate_alm(const DeltaPanel& panel, std::span<const double> cos_thetas, int lmax,
                      int mmax, const ScaleLadder& ladder = ScaleLadder::standard(),
                      std::uint64_t* step_counter = nullptr);

struct PartialAlm {
    AlmSet alm;
    std::vector<int> rings;
};

PartialAlm accumulate_alm_partial(const DeltaPanel& panel, std::span<const double> cos_thetas,
                                  int lmax, int mmax,
                                  const ScaleLadder& ladder = ScaleLadder::standard(),
                                  std::uint64_t* step_counter = nullptr);

AlmSet reduce_partials(std::span<const PartialAlm> parts, std::size_t n_rings);

SkyMap synthesis(const AlmSet& alm, const PixelGrid& grid, const TransformOptions& options = {});
AlmSet analysis(const SkyMap& map, int lmax, int mmax, const TransformOptions& options = {});

}  // namespace sht
