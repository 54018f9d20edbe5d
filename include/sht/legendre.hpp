// Drop-in Legendre-stage parameters (B200 build).  The recurrence itself runs inside the
// sm_100a kernels; only the ScaleLadder type of the reference's operator signatures
// (include/sht/legendre.hpp:26-36) and the host-side seeds are exposed here.
#pragma once

namespace sht {

// The 2^+-512 rescaling window of the reference.  The GPU kernels always track the standard
// ladder exactly; `unscaled()` (rescaling disabled) is accepted for API compatibility and
// gives identical results whenever the reference's unscaled run stays finite.
struct ScaleLadder {
    double step = 0x1p512;
    double inv_step = 0x1p-512;
    double hi = 0x1p512;
    double lo = 0x1p-512;
    bool enabled = true;

    static const ScaleLadder& standard();
    static const ScaleLadder& unscaled();
};

// log(mu_m) with glibc lgamma, the host-side precompute of every transform
double log_mu(int m);
// beta_lm = sqrt((4 l^2 - 1) / (l^2 - m^2)); std::domain_error at l == m
double beta_lm(int l, int m);

}  // namespace sht
