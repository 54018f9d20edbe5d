// Drop-in file containers (B200 build): the reference's SHTMAP1 / SHTALM1 formats
// (include/sht/io.hpp:9-17 of the reference): a text header ("key value" lines ending in
// "end") followed by little-endian float64 payload, so files interchange with the reference.
#pragma once

#include <string>

#include "sht/alm.hpp"

namespace sht {

void write_map(const std::string& path, const SkyMap& map);
SkyMap read_map(const std::string& path);
void write_alm(const std::string& path, const AlmSet& alm);
AlmSet read_alm(const std::string& path);

}  // namespace sht
