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
//   * the reference ladder is reproduced exactly at plan time: a scan runs every (order,
//     stream) through the reference's prefix (rescale when |Q| >= T_l = 2^512 / c_l, i.e.
//     |P mantissa| >= 2^512) and records the step where its scale k reaches 0 ("activation")
//     and the state (Q_{act-1}, Q_act) there.  Before activation the reference drops every
//     term, after it no rescale happens, so the kernels keep a lane at zero until its
//     activation step, inject the recorded state there and never test the ladder.  Tiles with
//     no activating stream are skipped; a tile's run starts at its first activation.
//   * persistent, warp-independent kernels: each warp pulls (order, tile of 32 x R
//     latitude-contiguous streams) items from a cost-sorted queue and stages the order's
//     coefficients (and c_l-scaled a_lm) in its own shared-memory slice LEG_CL degrees at a
//     time, so no block-wide barrier couples warps that sit in different phases.
//   * map2alm reduces over the 32 x R streams of a warp through a shared-memory transpose every
//     16 degrees and accumulates up to LEG_M2A_GROUP tiles per work item into a scratch slot;
//     a finalize kernel then sums each order's slots in a fixed order (one thread per
//     coefficient; no atomics on data, bitwise reproducible).

#include <atomic>
#include <climits>

#include "common.cuh"
#include "kernels.h"

namespace shtk {

namespace {
std::atomic<unsigned long long> g_launches{0};
}  // namespace
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
unsigned long long launch_count() { return g_launches.load(std::memory_order_relaxed); }

namespace {

constexpr double INV_LN2 = 1.4426950408889634074;  // legendre.cpp:10

#ifndef LEG_A2M_G
#define LEG_A2M_G 4  // alm2map FAST group: steps whose coefficients are loaded up front (with 4
                     // CTAs per SM: 6.80 ms at C4 against 6.83 ms for 8 at 3 CTAs per SM)
#endif
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

// Delta element (ring r, order index mi) of the alm2map output: in the local panel (delta +
// row_off[r]) or, on the fused exchange path, in ring r's owner's receive buffer (peer memory
// over NVLink); orders row_stride[r] apart (m-major exchange blocks) or contiguous
__device__ __forceinline__ double2* leg_out(const LegPlanView& p, double2* delta,
                                            const int64_t* __restrict__ row_off, int r, int mi) {
    double2* row = p.row_ptr ? p.row_ptr[r] : delta + row_off[r];
    return row + (p.row_stride ? (int64_t)mi * p.row_stride[r] : (int64_t)mi);
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
    count_launch();
}

// ---------------------------------------------------------------------------------------
// Plan: activation scan.  act = 0 for seeds already at k == 0, i for the step whose value
// brings k to 0, INT_MAX if the stream never reaches k == 0 (all terms dropped).
// ---------------------------------------------------------------------------------------
__global__ void leg_scan_kernel(LegPlanView p, int* __restrict__ act_out, double2* __restrict__ ck_out) {
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
    double2 ck = make_double2(0.0, act == 0 ? q1 : 0.0);  // state at activation (k == 0 scale)
    // unscaled ladder: the scale never changes, so a seed below k == 0 never counts
    bool done = !valid || k == 0 || p.unscaled;
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
                ck = make_double2(q1, q2);
            }
        }
        q0 = q1;
        q1 = q2;
    }
    if (valid) {
        act_out[(size_t)mi * p.st.n + s] = act;
        ck_out[(size_t)mi * p.st.n + s] = ck;
    }
}

void launch_leg_scan(const LegPlanView& p, int* act_dev, double2* ck_dev, cudaStream_t s) {
    dim3 grid((p.st.n + 127) / 128, p.n_m);
    leg_scan_kernel<<<grid, 128, 0, s>>>(p, act_dev, ck_dev);
    count_launch();
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
    count_launch();
}

// ---------------------------------------------------------------------------------------
// Persistent, warp-independent Legendre kernels.  Every warp pulls (order, tile) items from a
// cost-sorted queue and stages the order's coefficients (and c_l-scaled a_lm) for LEG_CL
// degrees at a time in its own shared-memory slice (no block barriers).
//
// Activation injection: a lane is zero (Q = 0, so it adds nothing) until its activation step
// act, where its state becomes the plan-time value (Q_{act-1}, Q_act) in the k == 0 scale --
// exactly the reference's state at the point its terms start to count.  The run of a tile
// starts at ic = i_s & ~1 (i_s = its first activation); steps up to the tile's last activation
// i_e test warp-uniformly for the next activation event, later steps are plain recurrence +
// accumulation.  No ladder check runs in the kernels.
// ---------------------------------------------------------------------------------------
namespace {

struct Coef {
    double A, ar, ai;  // recurrence coefficient, staged a_lm * c_l
};

// Per-warp staging, structure of arrays so a group of steps loads with 16-byte LDS.
struct __align__(16) CoefSoA {
    double A[LEG_CL];
    double ar[LEG_CL];
    double ai[LEG_CL];
    __device__ __forceinline__ void put(int j, const Coef& c) {
        A[j] = c.A;
        ar[j] = c.ar;
        ai[j] = c.ai;
    }
    __device__ __forceinline__ Coef get(int j) const { return Coef{A[j], ar[j], ai[j]}; }
};

__device__ __forceinline__ int warp_next_item(int* counter) {
    int it = 0;
    if ((threadIdx.x & 31) == 0) it = atomicAdd(counter, 1);
    return __shfl_sync(0xffffffffu, it, 0);
}

// next activation step after i over the warp's lanes and streams (INT_MAX: none)
template <int R>
__device__ __forceinline__ int next_activation(const int (&act)[R], int i) {
    int m = INT_MAX;
#pragma unroll
    for (int r = 0; r < R; ++r)
        if (act[r] > i) m = min(m, act[r]);
    return __reduce_min_sync(0xffffffffu, m);
}

// Activation steps kept in the warp's shared memory (column `lane` of a [S][32] array)
// instead of registers: they are read only at setup and in activation windows
// (map2alm: 8.08 -> 8.05 ms at C4 against keeping them in registers).
struct ActSmem {
    int* p;
    __device__ __forceinline__ int& operator[](int r) const { return p[r * 32]; }
};

template <int S>
__device__ __forceinline__ int next_activation(const ActSmem& act, int i) {
    int m = INT_MAX;
#pragma unroll
    for (int r = 0; r < S; ++r) {
        const int a = act[r];
        if (a > i) m = min(m, a);
    }
    return __reduce_min_sync(0xffffffffu, m);
}

// Lane setup shared by both kernels: zero state, activation steps, checkpoints staged in smem;
// seed lanes (act == 0) start from their checkpoint (0, P_mm).
// Lane k = q*R + r is stream r of tiles[q] (tiles[q] < 0: absent, its lanes stay zero).
template <int R, int NP, typename ActT>
__device__ __forceinline__ void lanes_setup(const LegPlanView& p, int mi, const int (&tiles)[NP], int lane,
                                            double (&x)[R * NP], double (&q0)[R * NP], double (&q1)[R * NP],
                                            ActT& act, double2 (*ck)[32]) {
#pragma unroll
    for (int k = 0; k < R * NP; ++k) {
        const int q = k / R, r = k % R;
        const int s = tiles[q] * (32 * R) + r * 32 + lane;
        x[k] = 0.0;
        q0[k] = q1[k] = 0.0;
        act[k] = INT_MAX;
        if (tiles[q] >= 0 && s < p.st.n) {
            const size_t o = (size_t)mi * p.st.n + s;
            x[k] = p.st.x[s];
            act[k] = p.ck_act[o];
            const double2 c = p.ck_q[o];
            ck[k][lane] = c;
            if (act[k] == 0) {
                q0[k] = c.x;
                q1[k] = c.y;
            }
        }
    }
}

template <int R>
struct A2MLane {
    double x[R], q0[R], q1[R];
    double2 ae[R], ao[R];  // even / odd degree-offset accumulators
    int act[R];  // (in shared memory, as map2alm keeps them, ptxas spills at the 128 cap)
};

// plain step: recurrence + accumulation
template <int R, bool ODD>
__device__ __forceinline__ void a2m_step(A2MLane<R>& L, const Coef& cf) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const double q2 = rec_step(cf.A, L.x[r], L.q1[r], L.q0[r]);
        double2& acc = ODD ? L.ao[r] : L.ae[r];
        acc.x = __fma_rn(cf.ar, q2, acc.x);
        acc.y = __fma_rn(cf.ai, q2, acc.y);
        L.q0[r] = L.q1[r];
        L.q1[r] = q2;
    }
}

// step i where some lanes activate: their (Q_{i-1}, Q_i) come from the checkpoint
template <int R, bool ODD>
__device__ __forceinline__ void a2m_step_act(A2MLane<R>& L, const Coef& cf, int i,
                                             const double2 (*ck)[32], int lane) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
        double q2 = rec_step(cf.A, L.x[r], L.q1[r], L.q0[r]);
        if (L.act[r] == i) {
            const double2 c = ck[r][lane];
            L.q1[r] = c.x;
            q2 = c.y;
        }
        double2& acc = ODD ? L.ao[r] : L.ae[r];
        acc.x = __fma_rn(cf.ar, q2, acc.x);
        acc.y = __fma_rn(cf.ai, q2, acc.y);
        L.q0[r] = L.q1[r];
        L.q1[r] = q2;
    }
}

}  // namespace

// A warp runs the NP tiles of one work item at once (S = R x NP streams per lane: the
// coefficient loads and the loop overhead of a step are shared by twice the streams at NP = 2).
template <int R, int NP>
__global__ void __launch_bounds__(LEG_WARPS * 32, LEG_A2M_MINB)
    leg_alm2map_kernel(LegPlanView p, const double2* __restrict__ alm, double2* __restrict__ delta,
                       const int64_t* __restrict__ row_off, int* __restrict__ counter) {
    constexpr int S = R * NP;
    struct WarpSmem {
        CoefSoA cf;
        double2 ck[S][32];
    };
    __shared__ WarpSmem sm_all[LEG_WARPS];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    CoefSoA& sm = sm_all[warp].cf;
    double2(*ck)[32] = sm_all[warp].ck;

    for (;;) {
        const int it = warp_next_item(counter);
        if (it >= p.n_a2m_items) return;
        const LegItem item = p.a2m_items[it];
        const int mi = item.mi;
        int tiles[NP];
        tiles[0] = item.a;
        if constexpr (NP > 1) tiles[1] = item.b;
        const int m = p.ms[mi];
        const int n = p.lmax - m;
        const int64_t toff = p.tab.tab_off[mi];
        const double* __restrict__ gA = p.tab.A + toff;
        const double* __restrict__ gC = p.tab.C + toff;
        const double2* __restrict__ galm = alm + alm_offset(m, p.lmax);
        int ic = INT_MAX, ie = -1;  // the run starts at the earliest tile start (0: seeds)
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            if (tiles[q] < 0) continue;
            const int2 info = p.tile_info[(size_t)mi * p.n_tiles + tiles[q]];
            ic = min(ic, leg_tile_start(info.x));
            ie = max(ie, info.y);
        }

        A2MLane<S> L;
        __syncwarp();
        lanes_setup<R, NP>(p, mi, tiles, lane, L.x, L.q0, L.q1, L.act, ck);
        const double2 a0 = galm[0];
#pragma unroll
        for (int r = 0; r < S; ++r) {
            // degree offset 0 term: a_mm P_mm (c_0 = 1) of lanes active from the seed
            L.ae[r] = make_double2(a0.x * L.q1[r], a0.y * L.q1[r]);
            L.ao[r] = make_double2(0.0, 0.0);
        }
        __syncwarp();
        int ev = next_activation<S>(L.act, ic - 1 + (ic == 0));  // ic == 0: seeds are set
        if (ic) {
            // the even step ic on its own, then (odd, even) pairs from ic + 1
            const double cc = gC[ic];
            const double2 v = galm[ic];
            const Coef c0{gA[ic], v.x * cc, v.y * cc};
            if (ic == ev) {
                a2m_step_act<S, false>(L, c0, ic, ck, lane);
                ev = next_activation<S>(L.act, ic);
            } else {
                a2m_step<S, false>(L, c0);
            }
        }
        const int i_first = ic + 1;

        // chunk c covers degree offsets i = i_first + c*CL .. ; lane j stages entry j.  The
        // raw loads are held in registers across the current chunk's steps; the c_l scaling
        // happens at staging time so no math waits on the prefetch.
        struct Raw {
            double A, C;
            double2 v;
        };
        constexpr int K = LEG_CL / 32;  // entries per lane per chunk
        auto fetch = [&](int c, Raw (&rw)[K]) {
#pragma unroll
            for (int q = 0; q < K; ++q) {
                const int i = i_first + c * LEG_CL + q * 32 + lane;
                if (i <= n) {
                    rw[q].C = gC[i];
                    rw[q].v = galm[i];
                    rw[q].A = gA[i];
                } else {
                    rw[q].A = rw[q].C = 0.0;
                    rw[q].v = make_double2(0.0, 0.0);
                }
            }
        };
        const int nchunks = (n - i_first + 1 + LEG_CL - 1) / LEG_CL;
        Raw nxt[K];
        if (nchunks > 0) fetch(0, nxt);
        for (int c = 0; c < nchunks; ++c) {
            __syncwarp();
#pragma unroll
            for (int q = 0; q < K; ++q)
                sm.put(q * 32 + lane, Coef{nxt[q].A, nxt[q].v.x * nxt[q].C, nxt[q].v.y * nxt[q].C});
            __syncwarp();
            if (c + 1 < nchunks) fetch(c + 1, nxt);
            const int i0 = i_first + c * LEG_CL;  // odd: pairs are (odd, even) degree offsets
            const int cnt = min(LEG_CL, n - i0 + 1);
            int j = 0;
            // activation window: pairs with a warp-uniform test for the next activation
            for (; j + 1 < cnt && i0 + j <= ie; j += 2) {
                const int i = i0 + j;
                const Coef c1 = sm.get(j), c2 = sm.get(j + 1);
                if (i == ev) {
                    a2m_step_act<S, true>(L, c1, i, ck, lane);
                    ev = next_activation<S>(L.act, i);
                } else {
                    a2m_step<S, true>(L, c1);
                }
                if (i + 1 == ev) {
                    a2m_step_act<S, false>(L, c2, i + 1, ck, lane);
                    ev = next_activation<S>(L.act, i + 1);
                } else {
                    a2m_step<S, false>(L, c2);
                }
            }
            // after the last activation: groups of 8 steps, coefficients loaded up front
            for (; j + LEG_A2M_G <= cnt; j += LEG_A2M_G) {
                Coef cg[LEG_A2M_G];
#pragma unroll
                for (int u = 0; u < LEG_A2M_G; u += 2) {
                    const double2 a = *reinterpret_cast<const double2*>(&sm.A[j + u]);
                    const double2 xr = *reinterpret_cast<const double2*>(&sm.ar[j + u]);
                    const double2 xi = *reinterpret_cast<const double2*>(&sm.ai[j + u]);
                    cg[u] = Coef{a.x, xr.x, xi.x};
                    cg[u + 1] = Coef{a.y, xr.y, xi.y};
                }
#pragma unroll
                for (int u = 0; u < LEG_A2M_G; u += 2) {
                    a2m_step<S, true>(L, cg[u]);
                    a2m_step<S, false>(L, cg[u + 1]);
                }
            }
            for (; j + 1 < cnt; j += 2) {
                a2m_step<S, true>(L, sm.get(j));
                a2m_step<S, false>(L, sm.get(j + 1));
            }
            if (j < cnt) {  // trailing odd step (last chunk only)
                const int i = i0 + j;
                if (i == ev) {
                    a2m_step_act<S, true>(L, sm.get(j), i, ck, lane);
                    ev = next_activation<S>(L.act, i);
                } else {
                    a2m_step<S, true>(L, sm.get(j));
                }
            }
        }

#pragma unroll
        for (int k = 0; k < S; ++k) {
            const int q = k / R, r = k % R;
            if (tiles[q] < 0) continue;
            const int s = tiles[q] * (32 * R) + r * 32 + lane;
            if (s >= p.st.n) continue;
            const double2 e = L.ae[k], o = L.ao[k];  // dead lanes stayed zero
            const int north = p.st.north[s], south = p.st.south[s];
            *leg_out(p, delta, row_off, north, mi) = cadd(e, o);
            if (south >= 0) *leg_out(p, delta, row_off, south, mi) = csub(e, o);
        }
    }
}

// Dead tiles: the reference writes exact zeros for streams that never reach k == 0.
// Threads over orders, one block row per tile: a thread reads its (order, tile) summary once
// and, when the tile is dead, writes the zeros of the tile's streams; consecutive threads write
// consecutive entries of a ring row (coalesced).  The earlier form -- threads over streams,
// one 16-byte entry per ring row each -- took 0.16 ms at C4 for ~170 MB of zeros.
__global__ void leg_zero_dead_kernel(LegPlanView p, double2* __restrict__ delta,
                                     const int64_t* __restrict__ row_off, int t0) {
    const int t = t0 + (int)blockIdx.y;
    const int mi = blockIdx.x * blockDim.x + threadIdx.x;
    if (mi >= p.n_m || p.tile_info[(size_t)mi * p.n_tiles + t].x >= 0) return;
    const double2 z = make_double2(0.0, 0.0);
    const int s_end = min(p.st.n, (t + 1) * LEG_TILE);
    for (int s = t * LEG_TILE; s < s_end; ++s) {
        *leg_out(p, delta, row_off, p.st.north[s], mi) = z;
        const int south = p.st.south[s];
        if (south >= 0) *leg_out(p, delta, row_off, south, mi) = z;
    }
}

int leg_persistent_blocks(int device) {
    static int cached[64] = {0};
    if (device >= 0 && device < 64 && cached[device]) return cached[device];
    int sms = 148, per = 1;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, leg_alm2map_kernel<LEG_R, LEG_A2M_P>, LEG_WARPS * 32, 0);
    const int v = sms * (per > 0 ? per : 1);
    if (device >= 0 && device < 64) cached[device] = v;
    return v;
}

void launch_leg_alm2map(const LegPlanView& p, const double2* alm, double2* delta,
                        const int64_t* row_off, int* counters, cudaStream_t s, int phases) {
    if (p.n_m == 0) return;
    if (phases & LEG_PHASE_ZERO) {
        for (int t0 = 0; t0 < p.n_tiles; t0 += 65535) {
            dim3 zg((p.n_m + 127) / 128, std::min(65535, p.n_tiles - t0));
            leg_zero_dead_kernel<<<zg, 128, 0, s>>>(p, delta, row_off, t0);
            count_launch();
        }
    }
    if (!(phases & LEG_PHASE_MAIN) || p.n_a2m_items == 0) return;
    int dev = 0;
    cudaGetDevice(&dev);
    int blocks = leg_persistent_blocks(dev);
    const int need = (p.n_a2m_items + LEG_WARPS - 1) / LEG_WARPS;
    if (need < blocks) blocks = need;
    if (!(phases & LEG_PHASE_NO_RESET)) cudaMemsetAsync(counters, 0, sizeof(int), s);
    leg_alm2map_kernel<LEG_R, LEG_A2M_P><<<blocks, LEG_WARPS * 32, 0, s>>>(p, alm, delta, row_off, counters);
    count_launch();
}

// ---------------------------------------------------------------------------------------
// map2alm: a_lm = c_l sum_r Delta^S_m(r) Q_lm(x_r), mirror paired
//
// A warp runs LEG_M2A_P tiles of one work item at once (S = LEG_R x LEG_M2A_P streams per
// lane): every lane sums its S streams per degree before the cross-lane reduction, so the
// shared-memory transpose -- which co-limited the kernel with the FP64 pipe at S = 4 (16
// STS.128 + 32 LDS.64 + 31 DADD per lane per 16 degrees, ~95% of the FP64 time in shared-
// memory wavefronts) -- is paid once per S x 16 stream-steps instead of once per 4 x 16.
// ---------------------------------------------------------------------------------------
namespace {

template <int S>
struct M2ALane {
    double x[S], q0[S], q1[S];
    double2 ds[S], dd[S];  // north+south / north-south ring Delta of the lane's streams
    ActSmem act;
};



__device__ __forceinline__ void m2a_load_d(double2& ds, double2& dd, int s, const LegPlanView& p,
                                           const double2* __restrict__ delta,
                                           const int64_t* __restrict__ row_off, int mi) {
    const double2 dn = delta[row_off[p.st.north[s]] + mi];
    const int south = p.st.south[s];
    if (south >= 0) {
        const double2 dso = delta[row_off[south] + mi];
        ds = cadd(dn, dso);
        dd = csub(dn, dso);
    } else {
        ds = dn;  // self-paired / unpaired row: alm_accumulate with dn (transforms.cpp:200-201)
        dd = dn;
    }
}

// One plain step; returns the lane's contribution (re, im) summed over its S streams.
template <int S, bool ODD>
__device__ __forceinline__ double2 m2a_step(M2ALane<S>& L, double A) {
    double2 part = make_double2(0.0, 0.0);
#pragma unroll
    for (int r = 0; r < S; ++r) {
        const double q2 = rec_step(A, L.x[r], L.q1[r], L.q0[r]);
        const double2 d = ODD ? L.dd[r] : L.ds[r];
        part.x = __fma_rn(d.x, q2, part.x);
        part.y = __fma_rn(d.y, q2, part.y);
        L.q0[r] = L.q1[r];
        L.q1[r] = q2;
    }
    return part;
}

// step i where some lanes activate (checkpointed (Q_{i-1}, Q_i))
template <int S, bool ODD>
__device__ __forceinline__ double2 m2a_step_act(M2ALane<S>& L, double A, int i, const double2 (*ck)[32],
                                                int lane) {
    double2 part = make_double2(0.0, 0.0);
#pragma unroll
    for (int r = 0; r < S; ++r) {
        double q2 = rec_step(A, L.x[r], L.q1[r], L.q0[r]);
        if (L.act[r] == i) {
            const double2 c = ck[r][lane];
            L.q1[r] = c.x;
            q2 = c.y;
        }
        const double2 d = ODD ? L.dd[r] : L.ds[r];
        part.x = __fma_rn(d.x, q2, part.x);
        part.y = __fma_rn(d.y, q2, part.y);
        L.q0[r] = L.q1[r];
        L.q1[r] = q2;
    }
    return part;
}

constexpr int M2A_G = 16;  // degrees per cross-lane reduction group
constexpr int M2A_S = LEG_R * LEG_M2A_P;

// Per-warp shared memory (dynamic: 4 warps x ~14 KB exceeds the 48 KB static limit)
struct M2AWarpSmem {
    double A[LEG_M2A_CL];
    double red[32][2 * M2A_G + 2];  // lane rows of (degree, re/im) partials, 16-byte aligned
    double2 ck[M2A_S][32];          // activation checkpoints of the current tiles
    int act[M2A_S][32];             // activation steps of the current tiles' streams
};

// Lanes of NP tiles at once: stream index q*R + r is stream r of tiles[q]; tiles[q] < 0 is an
// absent tile (its streams stay zero).  Seed lanes (act == 0) start from (0, P_mm).
template <int R, int NP>
__device__ __forceinline__ void m2a_lanes_setup(const LegPlanView& p, int mi, const int (&tiles)[NP],
                                                int lane, M2ALane<R * NP>& L, double2 (*ck)[32],
                                                const double2* __restrict__ delta,
                                                const int64_t* __restrict__ row_off) {
#pragma unroll
    for (int q = 0; q < NP; ++q) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int k = q * R + r;
            const int s = tiles[q] * (32 * R) + r * 32 + lane;
            L.x[k] = 0.0;
            L.q0[k] = L.q1[k] = 0.0;
            L.act[k] = INT_MAX;
            L.ds[k] = L.dd[k] = make_double2(0.0, 0.0);
            if (tiles[q] >= 0 && s < p.st.n) {
                const size_t o = (size_t)mi * p.st.n + s;
                L.x[k] = p.st.x[s];
                L.act[k] = p.ck_act[o];
                const double2 c = p.ck_q[o];
                ck[k][lane] = c;
                if (L.act[k] == 0) {
                    L.q0[k] = c.x;
                    L.q1[k] = c.y;
                }
                m2a_load_d(L.ds[k], L.dd[k], s, p, delta, row_off, mi);
            }
        }
    }
}

// One pass of a work item: NP of its tiles run together from the earliest start among them;
// the pass's per-degree sums go to the item's scratch slot (first pass stores, later passes
// add in place: a single lane owns each word, so the order is the pass order).
template <int R, int NP>
__device__ __forceinline__ void m2a_pass(const LegPlanView& p, const double2* __restrict__ delta,
                                         const int64_t* __restrict__ row_off, M2AWarpSmem& sm,
                                         int mi, int n, const double* __restrict__ gA,
                                         double2* __restrict__ part_out, const int (&tiles)[NP],
                                         bool first, int lane) {
    constexpr int S = R * NP;
    int ic = INT_MAX, ie = -1;
#pragma unroll
    for (int q = 0; q < NP; ++q) {
        if (tiles[q] < 0) continue;
        const int2 info = p.tile_info[(size_t)mi * p.n_tiles + tiles[q]];
        ic = min(ic, leg_tile_start(info.x));  // first step of the run (even; 0: seeds)
        ie = max(ie, info.y);
    }
    const int nchunks = (n + 1 - ic + LEG_M2A_CL - 1) / LEG_M2A_CL;  // degree offsets ic..n
    if (first)  // degrees below the first pass's start get no other first write
        for (int i = lane; i < ic; i += 32) part_out[i] = make_double2(0.0, 0.0);
    M2ALane<S> L;
    L.act.p = &sm.act[0][lane];
    __syncwarp();
    m2a_lanes_setup<R, NP>(p, mi, tiles, lane, L, sm.ck, delta, row_off);
    __syncwarp();
    int ev = next_activation<S>(L.act, ic - 1 + (ic == 0));

    constexpr int K = LEG_M2A_CL / 32;  // entries per lane per chunk
    auto fetch = [&](int c, double (&v)[K]) {
#pragma unroll
        for (int q = 0; q < K; ++q) {
            const int i = ic + c * LEG_M2A_CL + q * 32 + lane;
            v[q] = i <= n ? gA[i] : 0.0;
        }
    };
    // this lane's (degree, component) of the group in the scratch slot
    double* rmw_ptr = reinterpret_cast<double*>(part_out + ic) + lane;
    double nxt[K];
    fetch(0, nxt);
    for (int c = 0; c < nchunks; ++c) {
        __syncwarp();
#pragma unroll
        for (int q = 0; q < K; ++q) sm.A[q * 32 + lane] = nxt[q];
        __syncwarp();
        if (c + 1 < nchunks) fetch(c + 1, nxt);
        const int i0 = ic + c * LEG_M2A_CL;
        const int cnt = min(LEG_M2A_CL, n - i0 + 1);
        for (int g = 0; g < cnt; g += M2A_G) {
            const int gc = min(M2A_G, cnt - g);
            const int ig = i0 + g;  // even degree offset
            const int iw = ig + (lane >> 1);
            double* const wp = rmw_ptr;  // loop-carried: no per-group address rebuild
            rmw_ptr += 2 * M2A_G;
            // per-step lane contributions go straight to this lane's transpose row
            double2* const row = reinterpret_cast<double2*>(&sm.red[lane][0]);
            if ((ig > ie || (ev >= ig + M2A_G && ig > 0)) && gc == M2A_G) {
                // after the last activation: straight-line steps, coefficients in pairs; the
                // next pair's coefficients are loaded before this pair's partials are stored
                // (the compiler cannot move the load across the stores)
                double2 a = *reinterpret_cast<const double2*>(&sm.A[g]);
#pragma unroll
                for (int u = 0; u < M2A_G; u += 2) {
                    const double2 an = *reinterpret_cast<const double2*>(&sm.A[g + (u + 2 < M2A_G ? u + 2 : u)]);
                    row[u] = m2a_step<S, false>(L, a.x);
                    row[u + 1] = m2a_step<S, true>(L, a.y);
                    a = an;
                }
            } else {
                // activation window (warp-uniform event test per step), seed, partial group;
                // each step pair's coefficients are loaded one pair ahead (as in the FAST path)
                double2 anx = *reinterpret_cast<const double2*>(&sm.A[g]);
                for (int u = 0; u < M2A_G; u += 2) {
                    const int i = ig + u;
                    const double2 ap = anx;
                    if (u + 2 < M2A_G) anx = *reinterpret_cast<const double2*>(&sm.A[g + u + 2]);
                    double2 v1 = make_double2(0.0, 0.0), v2 = make_double2(0.0, 0.0);
                    if (u < gc) {
                        if (i == 0) {
                            // seed term (degree offset 0): no recurrence step
#pragma unroll
                            for (int r = 0; r < S; ++r) {
                                v1.x = __fma_rn(L.ds[r].x, L.q1[r], v1.x);
                                v1.y = __fma_rn(L.ds[r].y, L.q1[r], v1.y);
                            }
                        } else if (i == ev) {
                            v1 = m2a_step_act<S, false>(L, ap.x, i, sm.ck, lane);
                            ev = next_activation<S>(L.act, i);
                        } else {
                            v1 = m2a_step<S, false>(L, ap.x);
                        }
                        if (u + 1 < gc) {
                            if (i + 1 == ev) {
                                v2 = m2a_step_act<S, true>(L, ap.y, i + 1, sm.ck, lane);
                                ev = next_activation<S>(L.act, i + 1);
                            } else {
                                v2 = m2a_step<S, true>(L, ap.y);
                            }
                        }
                    }
                    row[u] = v1;
                    row[u + 1] = v2;
                }
            }
            // lane j reduces column j (degree ig + j/2, component j&1) over the 32 lane rows
            // in a fixed order (8 independent chains) and accumulates it into the slot
            __syncwarp();
            double s[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) s[k] = sm.red[k][lane];
#pragma unroll
            for (int rr = 8; rr < 32; rr += 8) {
#pragma unroll
                for (int k = 0; k < 8; ++k) s[k] += sm.red[rr + k][lane];
            }
            const double v = ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
            __syncwarp();
            if (iw <= n) {
                if (first) *wp = v;
                else asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(wp), "d"(v) : "memory");
            }
        }
    }
}

}  // namespace

template <int R>
__global__ void __launch_bounds__(LEG_WARPS * 32, LEG_M2A_MINB)
    leg_map2alm_kernel(LegPlanView p, const double2* __restrict__ delta,
                       const int64_t* __restrict__ row_off, int* __restrict__ queue,
                       double2* __restrict__ scratch) {
    static_assert(LEG_M2A_CL % M2A_G == 0, "chunk must hold whole reduction groups");
    extern __shared__ __align__(16) unsigned char m2a_smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    M2AWarpSmem& sm = reinterpret_cast<M2AWarpSmem*>(m2a_smem)[warp];

    for (;;) {
        const int it = warp_next_item(queue);
        if (it >= p.n_m2a_items) return;
        const LegItem item = p.m2a_items[it];
        const int mi = item.mi;
        const int m = p.ms[mi];
        const int n = p.lmax - m;
        const double* __restrict__ gA = p.tab.A + p.tab.tab_off[mi];
        double2* __restrict__ part_out = scratch + p.m2a_slot_base[mi] + (int64_t)item.g * (n + 1);
        int tt = 0;
        for (; tt + LEG_M2A_P <= item.b; tt += LEG_M2A_P) {
            int tiles[LEG_M2A_P];
#pragma unroll
            for (int q = 0; q < LEG_M2A_P; ++q) tiles[q] = p.tile_list[item.a + tt + q];
            m2a_pass<R, LEG_M2A_P>(p, delta, row_off, sm, mi, n, gA, part_out, tiles, tt == 0, lane);
        }
        for (; tt < item.b; ++tt) {  // leftover tiles one at a time
            const int tiles[1] = {p.tile_list[item.a + tt]};
            m2a_pass<R, 1>(p, delta, row_off, sm, mi, n, gA, part_out, tiles, tt == 0, lane);
        }
    }
}

// a_lm of order mi, degree offset i: the order's partial slots summed in slot order (batches
// of 4 loads), times c_l.  One thread per coefficient, after every item of the order is done.
__global__ void leg_m2a_finalize_kernel(LegPlanView p, const int* __restrict__ mis,
                                        const double2* __restrict__ scratch, double2* __restrict__ alm,
                                        int accumulate) {
    const int mi = mis ? mis[blockIdx.y] : (int)blockIdx.y;
    const int m = p.ms[mi];
    const int n = p.lmax - m;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i > n) return;
    const int G = p.m2a_items_per_m[mi];
    if (G == 0) return;  // no alive tile: the zero pass wrote it
    const double2* base = scratch + p.m2a_slot_base[mi] + i;
    double2 v = make_double2(0.0, 0.0);
    int g = 0;
    // batches of 8 slot loads in flight (the slots are summed in slot order either way)
    for (; g + 8 <= G; g += 8) {
        double2 a[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) a[u] = __ldcg(base + (int64_t)(g + u) * (n + 1));
#pragma unroll
        for (int u = 0; u < 8; ++u) v = cadd(v, a[u]);
    }
    for (; g + 4 <= G; g += 4) {
        const double2 a0 = __ldcg(base + (int64_t)g * (n + 1));
        const double2 a1 = __ldcg(base + (int64_t)(g + 1) * (n + 1));
        const double2 a2 = __ldcg(base + (int64_t)(g + 2) * (n + 1));
        const double2 a3 = __ldcg(base + (int64_t)(g + 3) * (n + 1));
        v = cadd(cadd(cadd(cadd(v, a0), a1), a2), a3);
    }
    for (; g < G; ++g) v = cadd(v, __ldcg(base + (int64_t)g * (n + 1)));
    const double c = p.tab.C[p.tab.tab_off[mi] + i];
    v = make_double2(v.x * c, v.y * c);
    double2* out = alm + alm_offset(m, p.lmax) + i;
    *out = accumulate ? cadd(*out, v) : v;
}

void launch_leg_m2a_finalize(const LegPlanView& p, const int* mis, int n_mis, const double2* scratch,
                             double2* alm, int accumulate, cudaStream_t s) {
    if (n_mis <= 0) return;
    dim3 grid((p.lmax + 1 + 127) / 128, n_mis);
    leg_m2a_finalize_kernel<<<grid, 128, 0, s>>>(p, mis, scratch, alm, accumulate);
    count_launch();
}

// orders without any alive tile: every term is dropped, a_lm = 0 (or unchanged when +=)
__global__ void leg_zero_orders_kernel(LegPlanView p, double2* __restrict__ alm) {
    const int mi = blockIdx.x;
    if (p.m2a_items_per_m[mi] > 0) return;
    const int m = p.ms[mi];
    double2* out = alm + alm_offset(m, p.lmax);
    for (int i = threadIdx.x; i <= p.lmax - m; i += blockDim.x) out[i] = make_double2(0.0, 0.0);
}

namespace {
constexpr size_t kM2ASmem = LEG_WARPS * sizeof(M2AWarpSmem);

// resident blocks per SM of the map2alm kernel (its dynamic shared memory opted in once per
// device)
int m2a_blocks_per_sm(int device) {
    static int cached[64] = {0};
    if (device >= 0 && device < 64 && cached[device]) return cached[device];
    cudaFuncSetAttribute(leg_map2alm_kernel<LEG_R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kM2ASmem);
    int per = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, leg_map2alm_kernel<LEG_R>, LEG_WARPS * 32, kM2ASmem);
    per = per > 0 ? per : 1;
    if (device >= 0 && device < 64) cached[device] = per;
    return per;
}
}  // namespace

int leg_m2a_warps(int device) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    return sms * m2a_blocks_per_sm(device) * LEG_WARPS;
}

void launch_leg_map2alm(const LegPlanView& p, const double2* delta, const int64_t* row_off,
                        double2* alm, int accumulate, int* counters, double2* scratch,
                        cudaStream_t s, int phases) {
    if (p.n_m == 0) return;
    if (!accumulate && (phases & LEG_PHASE_ZERO)) {
        leg_zero_orders_kernel<<<p.n_m, 128, 0, s>>>(p, alm);
        count_launch();
    }
    if (!(phases & LEG_PHASE_MAIN) || p.n_m2a_items == 0) return;
    int dev = 0;
    cudaGetDevice(&dev);
    int blocks = leg_m2a_warps(dev) / LEG_WARPS;
    const int need = (p.n_m2a_items + LEG_WARPS - 1) / LEG_WARPS;
    if (need < blocks) blocks = need;
    if (!(phases & LEG_PHASE_NO_RESET)) cudaMemsetAsync(counters, 0, sizeof(int), s);
    leg_map2alm_kernel<LEG_R><<<blocks, LEG_WARPS * 32, kM2ASmem, s>>>(p, delta, row_off, counters, scratch);
    count_launch();
    // whole launches reduce every order's slots here; pipelined band launches (defer_final)
    // leave them to the caller, which finalizes each order once its last launch is done
    if (!p.defer_final) launch_leg_m2a_finalize(p, nullptr, p.n_m, scratch, alm, accumulate, s);
}

}  // namespace shtk
