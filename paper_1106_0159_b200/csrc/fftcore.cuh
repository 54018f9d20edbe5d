// Small in-register DFT butterflies shared by the ring-FFT kernels (FP64, sign as a template
// parameter: S = -1 forward e^{-2 pi i jk/R}, S = +1 inverse, unnormalised).
#pragma once

#include "common.cuh"

namespace shtk {

template <int S>
__device__ __forceinline__ double2 mul_si(double2 a) {  // a * (S i)
    return S > 0 ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}

template <int S>
__device__ __forceinline__ void bfly4(double2& a0, double2& a1, double2& a2, double2& a3) {
    const double2 t0 = cadd(a0, a2), t1 = csub(a0, a2);
    const double2 t2 = cadd(a1, a3), t3 = mul_si<S>(csub(a1, a3));
    a0 = cadd(t0, t2);
    a2 = csub(t0, t2);
    a1 = cadd(t1, t3);
    a3 = csub(t1, t3);
}

// u[k] <- sum_j u[j] e^{S 2 pi i jk/R}, R in {2, 4, 8, 16}
template <int R, int S>
__device__ __forceinline__ void dft_pow2(double2 (&u)[R]) {
    constexpr double H = 0.70710678118654752440;
    if constexpr (R == 2) {
        const double2 a = u[0], b = u[1];
        u[0] = cadd(a, b);
        u[1] = csub(a, b);
    } else if constexpr (R == 4) {
        bfly4<S>(u[0], u[1], u[2], u[3]);
    } else if constexpr (R == 8) {
        double2 e0 = u[0], e1 = u[2], e2 = u[4], e3 = u[6];
        double2 o0 = u[1], o1 = u[3], o2 = u[5], o3 = u[7];
        bfly4<S>(e0, e1, e2, e3);
        bfly4<S>(o0, o1, o2, o3);
        o1 = cmul(o1, make_double2(H, S * H));
        o2 = mul_si<S>(o2);
        o3 = cmul(o3, make_double2(-H, S * H));
        u[0] = cadd(e0, o0);
        u[4] = csub(e0, o0);
        u[1] = cadd(e1, o1);
        u[5] = csub(e1, o1);
        u[2] = cadd(e2, o2);
        u[6] = csub(e2, o2);
        u[3] = cadd(e3, o3);
        u[7] = csub(e3, o3);
    } else if constexpr (R == 16) {
        // 16 = 4 x 4: DFT-4 over n2 (x[n1 + 4 n2]), twiddle W16^{n1 k1}, DFT-4 over n1,
        // output X[k1 + 4 k2] (register transpose at the end)
        constexpr double C1 = 0.92387953251128675613, S1 = 0.38268343236508977173;
#pragma unroll
        for (int n1 = 0; n1 < 4; ++n1) bfly4<S>(u[n1], u[n1 + 4], u[n1 + 8], u[n1 + 12]);
        // position n1 + 4 k1 now holds y[n1][k1]
        u[5] = cmul(u[5], make_double2(C1, S * S1));     // W^1
        u[9] = cmul(u[9], make_double2(H, S * H));       // W^2 (n1=1,k1=2)
        u[13] = cmul(u[13], make_double2(S1, S * C1));   // W^3
        u[6] = cmul(u[6], make_double2(H, S * H));       // W^2 (n1=2,k1=1)
        u[10] = mul_si<S>(u[10]);                        // W^4
        u[14] = cmul(u[14], make_double2(-H, S * H));    // W^6
        u[7] = cmul(u[7], make_double2(S1, S * C1));     // W^3 (n1=3,k1=1)
        u[11] = cmul(u[11], make_double2(-H, S * H));    // W^6
        u[15] = cmul(u[15], make_double2(-C1, -S * S1)); // W^9
#pragma unroll
        for (int k1 = 0; k1 < 4; ++k1) bfly4<S>(u[4 * k1], u[4 * k1 + 1], u[4 * k1 + 2], u[4 * k1 + 3]);
        // position 4 k1 + k2 holds X[k1 + 4 k2]: transpose the 4 x 4 index grid
        double2 x[16];
#pragma unroll
        for (int k1 = 0; k1 < 4; ++k1)
#pragma unroll
            for (int k2 = 0; k2 < 4; ++k2) x[k1 + 4 * k2] = u[4 * k1 + k2];
#pragma unroll
        for (int i = 0; i < 16; ++i) u[i] = x[i];
    }
}

}  // namespace shtk
