// Shared device helpers for the sm_100a SHT kernels (FP64 throughout).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace shtk {

__host__ __device__ __forceinline__ double2 cadd(double2 a, double2 b) {
    return make_double2(a.x + b.x, a.y + b.y);
}
__host__ __device__ __forceinline__ double2 csub(double2 a, double2 b) {
    return make_double2(a.x - b.x, a.y - b.y);
}
__host__ __device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__host__ __device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__host__ __device__ __forceinline__ double2 cscale(double2 a, double s) {
    return make_double2(a.x * s, a.y * s);
}
// multiply by s*i (s = +1 or -1)
__host__ __device__ __forceinline__ double2 cmul_si(double2 a, int s) {
    return s > 0 ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}

// AlmSet::offset (alm.hpp:27-30): m-major triangle.
__host__ __device__ __forceinline__ int64_t alm_offset(int m, int lmax) {
    const int64_t mm = m;
    return mm * (lmax + 1) - mm * (mm - 1) / 2;
}

}  // namespace shtk
