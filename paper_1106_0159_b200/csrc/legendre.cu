// Legendre stage of the spherical harmonic transform, hand-written for sm_100a (FP64).
//
// Reference algorithm (what these kernels reproduce, /root/reference/proj):
//   recurrence      PlmStream::advance            include/sht/legendre.hpp:106-113
//                   P_{m+1} = beta_0 x P_m ; P_l = beta x P_{l-1} - ratio P_{l-2}
//   seed            pmm_from_log                  src/legendre.cpp:62-76
//   scale ladder    plm_rescale (2^+-512 window)  include/sht/legendre.hpp:72-85
//   alm2map         detail::delta_a_columns_paired src/transforms.cpp:145-182
//                   terms kept only while the ladder scale k == 0 (transforms.cpp:27-32)
//   map2alm         detail::accumulate_columns_paired src/transforms.cpp:184-220
//
// B200 design:
//   * renormalised recurrence Q_l = P_l / c_l with c_l = (beta_l/beta_{l-1}) c_{l-2}, so a step
//     is Q_l = (A_l x) Q_{l-1} - Q_{l-2}: 1 DMUL + 1 DFMA, plus 2 DFMA to accumulate
//     (8 algorithmic flops in 4 FP64 pipe instructions).  c_l is folded into a_lm when it is
//     staged (alm2map) or applied once per l after the ring reduction (map2alm).
//   * the reference ladder is tracked exactly in the Q domain: a lane rescales when
//     |Q| >= T_l = 2^512 / c_l (== |P mantissa| >= 2^512) and its terms count from the step
//     where k reaches 0 ("activation").  A plan-time scan records the activation step of every
//     (order, stream); tiles whose streams never activate are skipped, steps before the first
//     activation of a tile run without accumulation, steps after the last activation run
//     without any check.
//   * block = one order m, W warps, each warp one tile of 32 x R latitude-contiguous streams;
//     recurrence coefficients and a_lm are staged through shared memory in double-buffered
//     chunks shared by the whole block.

#include <climits>

#include "common.cuh"
#include "kernels.h"

namespace shtk {

namespace {

constexpr double INV_LN2 = 1.4426950408889634074;  // legendre.cpp:10
constexpr double SCALE_DOWN = 0x1p-512;

__device__ __forceinline__ void seed_value(int m, double log_mu_m, double log2s2, int s2pos,
                                           double exp_lmu0, double& mant, int& k) {
    // pmm_from_log (legendre.cpp:62-76), evaluated with the same roundings (no contraction).
    if (m == 0) {
        mant = exp_lmu0;
        k = 0;
        return;
    }
    if (!s2pos) {
        mant = 0.0;
        k = 0;
        return;
    }
    const double e2 = __dadd_rn(__dmul_rn(log_mu_m, INV_LN2), __dmul_rn(0.5 * (double)m, log2s2));
    k = (int)floor(__dadd_rn(e2 / 512.0, 0.5));
    mant = exp2(__dsub_rn(e2, 512.0 * (double)k));
}

__device__ __forceinline__ double rec_step(double A, double x, double q1, double q0) {
    return __fma_rn(__dmul_rn(A, x), q1, -q0);
}

}  // namespace

// ---------------------------------------------------------------------------------------
// Plan: recurrence tables (one thread per order, sequential in l)
// ---------------------------------------------------------------------------------------
__global__ void leg_tables_kernel(const int* __restrict__ ms, int n_m, int lmax, LegTables tab) {
    const int mi = blockIdx.x * blockDim.x + threadIdx.x;
    if (mi >= n_m) return;
    const int m = ms[mi];
    const int n = lmax - m;
    double* A = tab.A + tab.tab_off[mi];
    double* C = tab.C + tab.tab_off[mi];
    double* T = tab.T + tab.tab_off[mi];
    const double dm = m;
    // beta_lm (legendre.cpp:22-27) with the reference's operation order.
    auto beta = [&](int l) {
        const double dl = l;
        return sqrt(__ddiv_rn(__dsub_rn(__dmul_rn(__dmul_rn(4.0, dl), dl), 1.0),
                             __dsub_rn(__dmul_rn(dl, dl), __dmul_rn(dm, dm))));
    };
    A[0] = 0.0;
    C[0] = 1.0;
    T[0] = 0x1p512;
    if (n >= 1) {
        const double b1 = beta(m + 1);
        A[1] = b1;
        C[1] = 1.0;
        T[1] = 0x1p512;
        double cm2 = 1.0, cm1 = 1.0, bprev = b1;
        for (int i = 2; i <= n; ++i) {
            const double b = beta(m + i);
            const double ratio = __ddiv_rn(b, bprev);  // RecurrenceCoeffs::build ratio[i]
            const double c = __dmul_rn(ratio, cm2);
            A[i] = __ddiv_rn(__dmul_rn(b, cm1), c);
            C[i] = c;
            T[i] = __ddiv_rn(0x1p512, c);
            cm2 = cm1;
            cm1 = c;
            bprev = b;
        }
    }
}

void launch_leg_tables(const int* ms_dev, int n_m, int lmax, LegTables tab, cudaStream_t s) {
    const int th = 64;
    leg_tables_kernel<<<(n_m + th - 1) / th, th, 0, s>>>(ms_dev, n_m, lmax, tab);
}

// ---------------------------------------------------------------------------------------
// Plan: activation scan.  act = 0 for seeds already at k == 0, i for the step whose value
// brings k to 0, INT_MAX if the stream never reaches k == 0 (all terms dropped).
// ---------------------------------------------------------------------------------------
__global__ void leg_scan_kernel(LegPlanView p, int* __restrict__ act_out) {
    const int mi = blockIdx.y;
    const int m = p.ms[mi];
    const int n = p.lmax - m;
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = s < p.st.n;
    double x = 0.0, q1 = 0.0, q0 = 0.0;
    int k = 0;
    if (valid) {
        x = p.st.x[s];
        seed_value(m, p.log_mu[m], p.st.log2s2[s], p.st.s2pos[s], p.exp_lmu0, q1, k);
    }
    int act = (valid && k == 0) ? 0 : INT_MAX;
    bool done = !valid || k == 0;
    const double* __restrict__ A = p.tab.A + p.tab.tab_off[mi];
    const double* __restrict__ T = p.tab.T + p.tab.tab_off[mi];
    for (int i = 1; i <= n; ++i) {
        if (__all_sync(0xffffffffu, done)) break;
        double q2 = rec_step(__ldg(A + i), x, q1, q0);
        if (!done && fabs(q2) >= __ldg(T + i)) {
            ++k;
            q2 *= SCALE_DOWN;
            q1 *= SCALE_DOWN;
            if (k == 0) {
                act = i;
                done = true;
            }
        }
        q0 = q1;
        q1 = q2;
    }
    if (valid) act_out[(size_t)mi * p.st.n + s] = act;
}

void launch_leg_scan(const LegPlanView& p, int* act_dev, cudaStream_t s) {
    dim3 grid((p.st.n + 127) / 128, p.n_m);
    leg_scan_kernel<<<grid, 128, 0, s>>>(p, act_dev);
}

__global__ void leg_tile_summary_kernel(LegPlanView p, const int* __restrict__ act,
                                        int2* __restrict__ info,
                                        unsigned long long* __restrict__ useful) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= p.n_m * p.n_tiles) return;
    const int mi = idx / p.n_tiles, t = idx % p.n_tiles;
    const int n = p.lmax - p.ms[mi];
    int is = INT_MAX, ie = -1;
    unsigned long long u = 0;
    for (int j = 0; j < LEG_TILE; ++j) {
        const int s = t * LEG_TILE + j;
        if (s >= p.st.n) break;
        const int a = act[(size_t)mi * p.st.n + s];
        if (a == INT_MAX) continue;
        is = min(is, a);
        ie = max(ie, a);
        u += (unsigned long long)(n - a + 1);
    }
    info[idx] = (ie < 0) ? make_int2(-1, -1) : make_int2(is, ie);
    if (u) atomicAdd(useful, u);
}

void launch_leg_tile_summary(const LegPlanView& p, const int* act_dev, int2* tile_info_dev,
                             unsigned long long* useful_dev, cudaStream_t s) {
    const int tot = p.n_m * p.n_tiles;
    leg_tile_summary_kernel<<<(tot + 127) / 128, 128, 0, s>>>(p, act_dev, tile_info_dev,
                                                              useful_dev);
}

// ---------------------------------------------------------------------------------------
// alm2map: Delta^A_m(r) = sum_l a_lm P_lm(x_r), mirror paired
// ---------------------------------------------------------------------------------------
namespace {

enum Phase { PREFIX = 0, CHECKED = 1, FAST = 2 };

template <int R>
struct A2MLane {
    double x[R], q0[R], q1[R];
    double2 ae[R], ao[R];  // even / odd degree offset accumulators
    int k[R];
};

// One recurrence step for all R streams of the lane; ODD selects the accumulator.
template <int R, int PH, bool ODD>
__device__ __forceinline__ void a2m_step(A2MLane<R>& L, double A, double T, double2 al) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
        double q2 = rec_step(A, L.x[r], L.q1[r], L.q0[r]);
        if (PH != FAST) {
            if (fabs(q2) >= T) {
                q2 *= SCALE_DOWN;
                L.q1[r] *= SCALE_DOWN;
                if (++L.k[r] == 0) {
                    // activation: every earlier term had k < 0 and is dropped by the reference
                    L.ae[r] = make_double2(0.0, 0.0);
                    L.ao[r] = make_double2(0.0, 0.0);
                }
            }
        }
        if (PH != PREFIX) {
            double2& acc = ODD ? L.ao[r] : L.ae[r];
            acc.x = __fma_rn(al.x, q2, acc.x);
            acc.y = __fma_rn(al.y, q2, acc.y);
        }
        L.q0[r] = L.q1[r];
        L.q1[r] = q2;
    }
}

template <int CL>
struct A2MStage {
    double A[2][CL];
    double T[2][CL];
    double2 al[2][CL];
};

}  // namespace

template <int R, int W, int CL>
__global__ void __launch_bounds__(W * 32)
    leg_alm2map_kernel(LegPlanView p, const double2* __restrict__ alm, double2* __restrict__ delta,
                       const int64_t* __restrict__ row_off) {
    __shared__ A2MStage<CL> sm;
    const int mi = p.m_order[blockIdx.x];
    const int m = p.ms[mi];
    const int n = p.lmax - m;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t toff = p.tab.tab_off[mi];
    const double* __restrict__ gA = p.tab.A + toff;
    const double* __restrict__ gC = p.tab.C + toff;
    const double* __restrict__ gT = p.tab.T + toff;
    const double2* __restrict__ galm = alm + alm_offset(m, p.lmax);
    const int tbeg = p.tile_list_off[mi], tcnt = p.tile_list_cnt[mi];
    const double lmu = p.log_mu[m];
    const int nchunks = (n + CL - 1) / CL;  // steps i = 1..n
    const double2 a0 = galm[0];

    for (int r0 = 0; r0 < tcnt; r0 += W) {
        const int ti = r0 + warp;
        const bool has = ti < tcnt;
        const int tile = has ? p.tile_list[tbeg + ti] : 0;
        const int2 info = has ? p.tile_info[(size_t)mi * p.n_tiles + tile] : make_int2(INT_MAX, -1);
        const int is = info.x, ie = info.y;

        A2MLane<R> L;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int s = tile * (32 * R) + r * 32 + lane;
            const bool valid = has && s < p.st.n;
            double mant = 0.0;
            int k = 0;
            double x = 0.0;
            if (valid) {
                x = p.st.x[s];
                seed_value(m, lmu, p.st.log2s2[s], p.st.s2pos[s], p.exp_lmu0, mant, k);
            }
            L.x[r] = x;
            L.q0[r] = 0.0;
            L.q1[r] = mant;
            L.k[r] = k;
            // degree offset 0 term: a_mm * P_mm (c_0 = 1), only when already at k == 0
            L.ae[r] = (k == 0) ? make_double2(a0.x * mant, a0.y * mant) : make_double2(0.0, 0.0);
            L.ao[r] = make_double2(0.0, 0.0);
        }
        bool fast_entered = false;

        // stage chunk 0
        if (nchunks > 0) {
            for (int j = threadIdx.x; j < CL; j += W * 32) {
                const int i = 1 + j;
                const bool in = i <= n;
                sm.A[0][j] = in ? gA[i] : 0.0;
                sm.T[0][j] = in ? gT[i] : 0x1p1000;
                if (in) {
                    const double c = gC[i];
                    const double2 v = galm[i];
                    sm.al[0][j] = make_double2(v.x * c, v.y * c);
                } else {
                    sm.al[0][j] = make_double2(0.0, 0.0);
                }
            }
        }
        __syncthreads();

        for (int c = 0; c < nchunks; ++c) {
            const int buf = c & 1;
            // prefetch chunk c+1 into registers
            constexpr int PER = (CL + W * 32 - 1) / (W * 32);
            double pA[PER], pT[PER];
            double2 pal[PER];
#pragma unroll
            for (int u = 0; u < PER; ++u) {
                const int j = threadIdx.x + u * W * 32;
                const int i = 1 + (c + 1) * CL + j;
                pA[u] = 0.0;
                pT[u] = 0x1p1000;
                pal[u] = make_double2(0.0, 0.0);
                if (j < CL && i <= n) {
                    pA[u] = gA[i];
                    pT[u] = gT[i];
                    const double cc = gC[i];
                    const double2 v = galm[i];
                    pal[u] = make_double2(v.x * cc, v.y * cc);
                }
            }

            if (has) {
                const int i0 = 1 + c * CL;
                const int cnt = min(CL, n - i0 + 1);
                int j = 0;
                for (; j + 1 < cnt; j += 2) {
                    const int i = i0 + j;  // odd degree offset, i+1 even
                    const double A1 = sm.A[buf][j], A2 = sm.A[buf][j + 1];
                    const double2 l1 = sm.al[buf][j], l2 = sm.al[buf][j + 1];
                    if (i + 1 < is) {
                        const double T1 = sm.T[buf][j], T2 = sm.T[buf][j + 1];
                        a2m_step<R, PREFIX, true>(L, A1, T1, l1);
                        a2m_step<R, PREFIX, false>(L, A2, T2, l2);
                    } else if (i > ie) {
                        if (!fast_entered) {
                            fast_entered = true;
#pragma unroll
                            for (int r = 0; r < R; ++r)
                                if (L.k[r] != 0) L.q0[r] = L.q1[r] = 0.0;  // dead lanes
                        }
                        a2m_step<R, FAST, true>(L, A1, 0.0, l1);
                        a2m_step<R, FAST, false>(L, A2, 0.0, l2);
                    } else {
                        const double T1 = sm.T[buf][j], T2 = sm.T[buf][j + 1];
                        a2m_step<R, CHECKED, true>(L, A1, T1, l1);
                        a2m_step<R, CHECKED, false>(L, A2, T2, l2);
                    }
                }
                if (j < cnt) {  // trailing odd step (last chunk only)
                    const int i = i0 + j;
                    const double A1 = sm.A[buf][j], T1 = sm.T[buf][j];
                    const double2 l1 = sm.al[buf][j];
                    if (i > ie && fast_entered)
                        a2m_step<R, FAST, true>(L, A1, 0.0, l1);
                    else
                        a2m_step<R, CHECKED, true>(L, A1, T1, l1);
                }
            }

            // publish the prefetched chunk into the other buffer
#pragma unroll
            for (int u = 0; u < PER; ++u) {
                const int j = threadIdx.x + u * W * 32;
                if (j < CL && c + 1 < nchunks) {
                    sm.A[buf ^ 1][j] = pA[u];
                    sm.T[buf ^ 1][j] = pT[u];
                    sm.al[buf ^ 1][j] = pal[u];
                }
            }
            __syncthreads();
        }

        if (has) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int s = tile * (32 * R) + r * 32 + lane;
                if (s >= p.st.n) continue;
                double2 e = L.ae[r], o = L.ao[r];
                if (L.k[r] != 0) e = o = make_double2(0.0, 0.0);
                const int north = p.st.north[s], south = p.st.south[s];
                delta[row_off[north] + mi] = cadd(e, o);
                if (south >= 0) delta[row_off[south] + mi] = csub(e, o);
            }
        }
    }
}

// Dead tiles: the reference writes exact zeros for streams that never reach k == 0.
__global__ void leg_zero_dead_kernel(LegPlanView p, double2* __restrict__ delta,
                                     const int64_t* __restrict__ row_off) {
    const int mi = blockIdx.y;
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= p.st.n) return;
    const int t = s / LEG_TILE;
    if (p.tile_info[(size_t)mi * p.n_tiles + t].x >= 0) return;
    const double2 z = make_double2(0.0, 0.0);
    delta[row_off[p.st.north[s]] + mi] = z;
    const int south = p.st.south[s];
    if (south >= 0) delta[row_off[south] + mi] = z;
}

void launch_leg_alm2map(const LegPlanView& p, const double2* alm, double2* delta,
                        const int64_t* row_off, cudaStream_t s) {
    if (p.n_m == 0) return;
    dim3 zg((p.st.n + 127) / 128, p.n_m);
    leg_zero_dead_kernel<<<zg, 128, 0, s>>>(p, delta, row_off);
    leg_alm2map_kernel<LEG_R, LEG_W, 64><<<p.n_m, LEG_W * 32, 0, s>>>(p, alm, delta, row_off);
}

// ---------------------------------------------------------------------------------------
// map2alm: a_lm = sum_r Delta^S_m(r) P_lm(x_r), mirror paired
// ---------------------------------------------------------------------------------------
namespace {

template <int R>
struct M2ALane {
    double x[R], q0[R], q1[R];
    double2 ds[R], dd[R];  // masked (zero until activation) north+south / north-south
    int k[R];
};

template <int R>
__device__ __forceinline__ void m2a_load_d(M2ALane<R>& L, int r, int s, const LegPlanView& p,
                                           const double2* __restrict__ delta,
                                           const int64_t* __restrict__ row_off, int mi) {
    const double2 dn = delta[row_off[p.st.north[s]] + mi];
    const int south = p.st.south[s];
    if (south >= 0) {
        const double2 dsouth = delta[row_off[south] + mi];
        L.ds[r] = cadd(dn, dsouth);
        L.dd[r] = csub(dn, dsouth);
    } else {
        L.ds[r] = dn;  // self-paired / unpaired row: alm_accumulate with dn (transforms.cpp:200-201)
        L.dd[r] = dn;
    }
}

// One step; returns the lane's contribution (re, im) summed over its R streams.
template <int R, int PH, bool ODD>
__device__ __forceinline__ double2 m2a_step(M2ALane<R>& L, double A, double T, const LegPlanView& p,
                                            const double2* __restrict__ delta,
                                            const int64_t* __restrict__ row_off, int mi,
                                            int tile, int lane) {
    double2 part = make_double2(0.0, 0.0);
#pragma unroll
    for (int r = 0; r < R; ++r) {
        double q2 = rec_step(A, L.x[r], L.q1[r], L.q0[r]);
        if (PH != FAST) {
            if (fabs(q2) >= T) {
                q2 *= SCALE_DOWN;
                L.q1[r] *= SCALE_DOWN;
                if (++L.k[r] == 0) {
                    const int s = tile * (32 * R) + r * 32 + lane;
                    m2a_load_d<R>(L, r, s, p, delta, row_off, mi);
                }
            }
        }
        if (PH != PREFIX) {
            const double2 d = ODD ? L.dd[r] : L.ds[r];
            part.x = __fma_rn(d.x, q2, part.x);
            part.y = __fma_rn(d.y, q2, part.y);
        }
        L.q0[r] = L.q1[r];
        L.q1[r] = q2;
    }
    return part;
}

template <int W, int CL>
struct M2AStage {
    double A[2][CL];
    double T[2][CL];
    double C[2][CL];
    double red[W][32][17];      // per-warp lane transpose
    double res[2][W][CL][2];    // per-warp reduced chunk results
};

}  // namespace

template <int R, int W, int CL>
__global__ void __launch_bounds__(W * 32)
    leg_map2alm_kernel(LegPlanView p, const double2* __restrict__ delta,
                       const int64_t* __restrict__ row_off, double2* __restrict__ alm,
                       int accumulate) {
    static_assert(CL % 8 == 0, "chunk must hold whole 8-step reduction groups");
    extern __shared__ __align__(16) unsigned char smraw[];
    M2AStage<W, CL>& sm = *reinterpret_cast<M2AStage<W, CL>*>(smraw);
    const int mi = p.m_order[blockIdx.x];
    const int m = p.ms[mi];
    const int n = p.lmax - m;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t toff = p.tab.tab_off[mi];
    const double* __restrict__ gA = p.tab.A + toff;
    const double* __restrict__ gC = p.tab.C + toff;
    const double* __restrict__ gT = p.tab.T + toff;
    double2* __restrict__ out = alm + alm_offset(m, p.lmax);
    const int tbeg = p.tile_list_off[mi], tcnt = p.tile_list_cnt[mi];
    const double lmu = p.log_mu[m];
    const int nchunks = (n + 1 + CL - 1) / CL;  // steps i = 0..n

    if (tcnt == 0) {  // every stream of this order is dropped: a_lm = 0 (or unchanged)
        if (!accumulate)
            for (int i = threadIdx.x; i <= n; i += W * 32) out[i] = make_double2(0.0, 0.0);
        return;
    }

    for (int r0 = 0; r0 < tcnt; r0 += W) {
        const bool first_round = (r0 == 0);
        const int ti = r0 + warp;
        const bool has = ti < tcnt;
        const int tile = has ? p.tile_list[tbeg + ti] : 0;
        const int2 info = has ? p.tile_info[(size_t)mi * p.n_tiles + tile] : make_int2(INT_MAX, -1);
        const int is = info.x, ie = info.y;

        M2ALane<R> L;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int s = tile * (32 * R) + r * 32 + lane;
            const bool valid = has && s < p.st.n;
            double mant = 0.0, x = 0.0;
            int k = 1;  // invalid lanes: never active
            if (valid) {
                x = p.st.x[s];
                seed_value(m, lmu, p.st.log2s2[s], p.st.s2pos[s], p.exp_lmu0, mant, k);
            }
            L.x[r] = x;
            L.q0[r] = 0.0;
            L.q1[r] = valid ? mant : 0.0;
            L.k[r] = k;
            L.ds[r] = L.dd[r] = make_double2(0.0, 0.0);
            if (valid && k == 0) m2a_load_d<R>(L, r, s, p, delta, row_off, mi);
        }
        bool fast_entered = false;

        // stage chunk 0 (degree offsets 0..CL-1)
        for (int j = threadIdx.x; j < CL; j += W * 32) {
            const bool in = j <= n;
            sm.A[0][j] = in ? gA[j] : 0.0;
            sm.T[0][j] = in ? gT[j] : 0x1p1000;
            sm.C[0][j] = in ? gC[j] : 0.0;
        }
        __syncthreads();

        for (int c = 0; c < nchunks; ++c) {
            const int buf = c & 1;
            constexpr int PER = (CL + W * 32 - 1) / (W * 32);
            double pA[PER], pT[PER], pC[PER];
#pragma unroll
            for (int u = 0; u < PER; ++u) {
                const int j = threadIdx.x + u * W * 32;
                const int i = (c + 1) * CL + j;
                const bool in = j < CL && i <= n;
                pA[u] = in ? gA[i] : 0.0;
                pT[u] = in ? gT[i] : 0x1p1000;
                pC[u] = in ? gC[i] : 0.0;
            }
            // reduce the previous chunk's per-warp results (fixed warp order) into a_lm
            if (c > 0) {
                for (int t = threadIdx.x; t < 2 * CL; t += W * 32) {
                    const int j = t >> 1, comp = t & 1;
                    const int i = (c - 1) * CL + j;
                    if (i <= n) {
                        double v = 0.0;
#pragma unroll
                        for (int w = 0; w < W; ++w) v += sm.res[buf ^ 1][w][j][comp];
                        v *= sm.C[buf ^ 1][j];
                        double* o = reinterpret_cast<double*>(out + i) + comp;
                        *o = (first_round && !accumulate) ? v : *o + v;
                    }
                }
            }

            const int i0 = c * CL;
            const int cnt = min(CL, n - i0 + 1);
            for (int g = 0; g < CL; g += 8) {
                double part[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) part[u] = 0.0;
                bool any = false;
                if (has && g < cnt) {
#pragma unroll
                    for (int u = 0; u < 8; u += 2) {
                        const int j = g + u;
                        if (j >= cnt) break;
                        const int i = i0 + j;  // even degree offset
                        const double A1 = sm.A[buf][j], T1 = sm.T[buf][j];
                        const bool two = j + 1 < cnt;
                        const double A2 = two ? sm.A[buf][j + 1] : 0.0;
                        const double T2 = two ? sm.T[buf][j + 1] : 0x1p1000;
                        double2 c1 = make_double2(0.0, 0.0), c2 = make_double2(0.0, 0.0);
                        if (i == 0) {
                            // seed term (degree offset 0): no recurrence step
#pragma unroll
                            for (int r = 0; r < R; ++r) {
                                c1.x = __fma_rn(L.ds[r].x, L.q1[r], c1.x);
                                c1.y = __fma_rn(L.ds[r].y, L.q1[r], c1.y);
                            }
                            any = true;
                            if (two) {
                                if (1 > ie && !fast_entered) {
                                    fast_entered = true;
#pragma unroll
                                    for (int r = 0; r < R; ++r)
                                        if (L.k[r] != 0) {
                                            L.q0[r] = L.q1[r] = 0.0;
                                            L.ds[r] = L.dd[r] = make_double2(0.0, 0.0);
                                        }
                                }
                                if (fast_entered)
                                    c2 = m2a_step<R, FAST, true>(L, A2, T2, p, delta, row_off, mi, tile, lane);
                                else
                                    c2 = m2a_step<R, CHECKED, true>(L, A2, T2, p, delta, row_off, mi, tile, lane);
                            }
                        } else if (i + 1 < is) {
                            m2a_step<R, PREFIX, false>(L, A1, T1, p, delta, row_off, mi, tile, lane);
                            if (two) m2a_step<R, PREFIX, true>(L, A2, T2, p, delta, row_off, mi, tile, lane);
                        } else if (i > ie) {
                            if (!fast_entered) {
                                fast_entered = true;
#pragma unroll
                                for (int r = 0; r < R; ++r)
                                    if (L.k[r] != 0) {
                                        L.q0[r] = L.q1[r] = 0.0;
                                        L.ds[r] = L.dd[r] = make_double2(0.0, 0.0);
                                    }
                            }
                            any = true;
                            c1 = m2a_step<R, FAST, false>(L, A1, T1, p, delta, row_off, mi, tile, lane);
                            if (two) c2 = m2a_step<R, FAST, true>(L, A2, T2, p, delta, row_off, mi, tile, lane);
                        } else {
                            any = true;
                            c1 = m2a_step<R, CHECKED, false>(L, A1, T1, p, delta, row_off, mi, tile, lane);
                            if (two) c2 = m2a_step<R, CHECKED, true>(L, A2, T2, p, delta, row_off, mi, tile, lane);
                        }
                        part[2 * u + 0] = c1.x;
                        part[2 * u + 1] = c1.y;
                        part[2 * u + 2] = c2.x;
                        part[2 * u + 3] = c2.y;
                    }
                }
                // reduce the 16 values over the 32 lanes of the warp (fixed order)
                double v = 0.0;
                if (__any_sync(0xffffffffu, any)) {
#pragma unroll
                    for (int u = 0; u < 16; ++u) sm.red[warp][lane][u] = part[u];
                    __syncwarp();
                    const int col = lane & 15, half = lane >> 4;
#pragma unroll
                    for (int row = 0; row < 16; ++row) v += sm.red[warp][half * 16 + row][col];
                    v += __shfl_xor_sync(0xffffffffu, v, 16);
                    __syncwarp();
                }
                if (lane < 16) sm.res[buf][warp][g + (lane >> 1)][lane & 1] = v;
            }

#pragma unroll
            for (int u = 0; u < PER; ++u) {
                const int j = threadIdx.x + u * W * 32;
                if (j < CL && c + 1 < nchunks) {
                    sm.A[buf ^ 1][j] = pA[u];
                    sm.T[buf ^ 1][j] = pT[u];
                    sm.C[buf ^ 1][j] = pC[u];
                }
            }
            __syncthreads();
        }
        // reduce the final chunk
        {
            const int c = nchunks;
            const int buf = c & 1;
            for (int t = threadIdx.x; t < 2 * CL; t += W * 32) {
                const int j = t >> 1, comp = t & 1;
                const int i = (c - 1) * CL + j;
                if (i <= n) {
                    double v = 0.0;
#pragma unroll
                    for (int w = 0; w < W; ++w) v += sm.res[buf ^ 1][w][j][comp];
                    v *= sm.C[buf ^ 1][j];
                    double* o = reinterpret_cast<double*>(out + i) + comp;
                    *o = (first_round && !accumulate) ? v : *o + v;
                }
            }
        }
        __syncthreads();
    }
}

void launch_leg_map2alm(const LegPlanView& p, const double2* delta, const int64_t* row_off,
                        double2* alm, int accumulate, cudaStream_t s) {
    if (p.n_m == 0) return;
    constexpr int CL = 64;
    const size_t smem = sizeof(M2AStage<LEG_W, CL>);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(leg_map2alm_kernel<LEG_R, LEG_W, CL>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    leg_map2alm_kernel<LEG_R, LEG_W, CL><<<p.n_m, LEG_W * 32, smem, s>>>(p, delta, row_off, alm,
                                                                         accumulate);
}

}  // namespace shtk
