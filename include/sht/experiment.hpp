// Drop-in synthetic inputs (B200 build): the reference's counter-based generators
// (include/sht/experiment.hpp:14-28), host side.
#pragma once

#include <cstdint>

#include "sht/alm.hpp"

namespace sht {

std::uint64_t splitmix64_at(std::uint64_t seed, std::uint64_t index);
double uniform_pm1(std::uint64_t seed, std::uint64_t index);
AlmSet random_alm(int lmax, int mmax, std::uint64_t seed);
double roundtrip_error(const AlmSet& a_init, const AlmSet& a_out);

}  // namespace sht
