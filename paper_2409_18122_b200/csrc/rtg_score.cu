// rtg_score.cu -- scoring kernels.
//
// Phase A (collision, a4): first colliding waypoint per trajectory.
//   dense : every waypoint x every collidable Gaussian, TMA-bulk-staged record tiles in smem,
//           split over the Gaussian axis (integer atomicMin / flag stores: order-free).
//   culled: one warp per trajectory walks t = 0..T-1 and stops at the first collision
//           (early exit); each waypoint tests only the collision-grid cells within the
//           largest bounding radius, lanes load-balanced over the union of cell rows.
// Phase B (visibility + gain, a5) over the info waypoints of feasible trajectories
//   (two-phase; or of all trajectories with RTG_SCORE_FULL_GAIN):
//   dense : waypoints in registers (4 per thread) x TMA-staged Gaussian tiles.
//   culled: one warp per waypoint enumerates the visibility-grid columns under the frustum's
//           footprint; whole z-cell runs strictly inside the frustum are added from exact
//           fixed-point prefix sums, the straddling cells' Gaussians are tested one by one.
// Reduction (a6) per trajectory and argmax (a7).
#include <algorithm>
#include <cfloat>
#include <cmath>

#include "rtg_host.hpp"

namespace rtg {

constexpr unsigned kFull = 0xffffffffu;

// ===================================================================== dense phase A
// Each thread owns 2 waypoints of the flattened K*T index; blockIdx.y splits the Gaussians.
constexpr int kDenseColThreads = 256;
#ifndef RTG_DENSE_COL_WPT
#define RTG_DENSE_COL_WPT 4
#endif
constexpr int kDenseColWpt = RTG_DENSE_COL_WPT;

__global__ void __launch_bounds__(kDenseColThreads) k_col_dense(
    const float* __restrict__ X, const float* __restrict__ Y, const float* __restrict__ Zw, int K, int T,
    const CRec* __restrict__ crec, const CMat* __restrict__ cmat, const CSrc* __restrict__ csrc, const rtg_robot rb,
    long long n_col_pad, int tiles_per_split, float gq, int* __restrict__ first_col,
    unsigned char* __restrict__ wp_col, int all_waypoints, unsigned long long* __restrict__ stats) {
    __shared__ __align__(128) CRec s_tile[2][kTile];
    __shared__ __align__(8) uint64_t s_bar[2];
    const long long KT = (long long)K * T;
    const long long tile0 = (long long)blockIdx.y * tiles_per_split;
    const long long ntiles_all = n_col_pad / kTile;
    long long ntiles = ntiles_all - tile0;
    if (ntiles > tiles_per_split) ntiles = tiles_per_split;
    if (ntiles <= 0) return;

    float px[kDenseColWpt], py[kDenseColWpt], pz[kDenseColWpt];
    int kk[kDenseColWpt], tt[kDenseColWpt];
    bool act[kDenseColWpt], hit[kDenseColWpt];
#pragma unroll
    for (int j = 0; j < kDenseColWpt; ++j) {
        long long i = (long long)blockIdx.x * (kDenseColThreads * kDenseColWpt) + j * kDenseColThreads + threadIdx.x;
        act[j] = i < KT;
        hit[j] = false;
        long long ii = act[j] ? i : 0;
        px[j] = X[ii]; py[j] = Y[ii]; pz[j] = Zw[ii];
        act[j] = act[j] && isfinite(px[j]) && isfinite(py[j]) && isfinite(pz[j]);
        kk[j] = (int)(ii / T);
        tt[j] = (int)(ii % T);
    }
    static_assert(kDenseColWpt % 2 == 0, "waypoints go in pairs (packed FP32)");
    unsigned long long P2x[kDenseColWpt / 2], P2y[kDenseColWpt / 2], P2z[kDenseColWpt / 2];
#pragma unroll
    for (int j = 0; j < kDenseColWpt; j += 2) {
        P2x[j / 2] = f2_pack(px[j], px[j + 1]);
        P2y[j / 2] = f2_pack(py[j], py[j + 1]);
        P2z[j / 2] = f2_pack(pz[j], pz[j + 1]);
    }
    if (threadIdx.x == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const uint32_t tile_bytes = kTile * sizeof(CRec);
    if (threadIdx.x == 0) {
        for (int s = 0; s < 2 && s < ntiles; ++s) {
            mbar_expect_tx(&s_bar[s], tile_bytes);
            bulk_g2s(s_tile[s], crec + (tile0 + s) * kTile, tile_bytes, &s_bar[s]);
        }
    }
    unsigned nref = 0;
    for (long long it = 0; it < ntiles; ++it) {
        const int s = (int)(it & 1);
        // opportunistic skip: a waypoint after a known collision cannot change first_col
        bool live = false;
#pragma unroll
        for (int j = 0; j < kDenseColWpt; ++j) {
            if (act[j] && !hit[j] && !all_waypoints) {
                int fc = *((volatile int*)&first_col[kk[j]]);
                if (fc < tt[j]) act[j] = false;
            }
            live |= act[j] && !hit[j];
        }
        mbar_wait(&s_bar[s], (uint32_t)((it >> 1) & 1));
        if (__syncthreads_or(live)) {
            const CRec* tile = s_tile[s];
#pragma unroll 4
            for (int g = 0; g < kTile; ++g) {
                const CRec A = tile[g];
                float dxs[kDenseColWpt], dys[kDenseColWpt], dzs[kDenseColWpt], d2s[kDenseColWpt];
#pragma unroll
                for (int j = 0; j < kDenseColWpt; j += 2) {
                    // two waypoints in one register pair (packed FP32, each half rounds like the
                    // scalar d = p - mu, d2 = fma(dx, dx, fma(dy, dy, dz * dz)))
                    const unsigned long long DX = f2_sub(P2x[j / 2], f2_pack(A.x, A.x));
                    const unsigned long long DY = f2_sub(P2y[j / 2], f2_pack(A.y, A.y));
                    const unsigned long long DZ = f2_sub(P2z[j / 2], f2_pack(A.z, A.z));
                    const unsigned long long D2 = f2_fma(DX, DX, f2_fma(DY, DY, f2_mul(DZ, DZ)));
                    f2_unpack(DX, dxs[j], dxs[j + 1]);
                    f2_unpack(DY, dys[j], dys[j + 1]);
                    f2_unpack(DZ, dzs[j], dzs[j + 1]);
                    f2_unpack(D2, d2s[j], d2s[j + 1]);
                }
                bool near = false;
#pragma unroll
                for (int j = 0; j < kDenseColWpt; ++j) near |= d2s[j] < A.rb2 && act[j] && !hit[j];
                if (near) {   // inside some waypoint's bounding sphere: the full test (rare)
                    const long long gi = (tile0 + it) * kTile + g;
#pragma unroll
                    for (int j = 0; j < kDenseColWpt; ++j) {
                        if (d2s[j] < A.rb2 && act[j] && !hit[j])
                            hit[j] = collide_full(cmat[gi].m, dxs[j], dys[j], dzs[j], gq, &csrc[gi], rb, px[j], py[j],
                                                  pz[j], A.x, A.y, A.z, nref);
                    }
                }
            }
        } else {
            // nothing left to test in this block: drain the in-flight copies and stop
            __syncthreads();
            if (threadIdx.x == 0 && it + 1 < ntiles) mbar_wait(&s_bar[s ^ 1], (uint32_t)(((it + 1) >> 1) & 1));
            break;
        }
        __syncthreads();
        if (threadIdx.x == 0 && it + 2 < ntiles) {
            mbar_expect_tx(&s_bar[s], tile_bytes);
            bulk_g2s(s_tile[s], crec + (tile0 + it + 2) * kTile, tile_bytes, &s_bar[s]);
        }
    }
#pragma unroll
    for (int j = 0; j < kDenseColWpt; ++j) {
        if (hit[j]) {
            long long i = (long long)kk[j] * T + tt[j];
            if (wp_col) wp_col[i] = 1;
            atomicMin(&first_col[kk[j]], tt[j]);
        }
    }
    if (stats && nref) atomicAdd(&stats[0], (unsigned long long)nref);
}

// ===================================================================== culled phase A
constexpr int kWarps = 8;   // warps per block of the persistent culled kernels

// work item e = (chunk c, trajectory k), chunk-major: waypoints c*kColChunk .. +kColChunk-1 of k,
// t ascending, stopping at the chunk's first collision; first_col[k] (preset to T) = atomicMin of
// the chunks' first collisions, so it is the first collision of k whatever the schedule.  A chunk
// whose trajectory already collided earlier is skipped (chunk-major order: chunk c - 1 of every
// trajectory was handed out before chunk c), so the early exit of a4 survives the split while the
// long collision-free trajectories no longer serialise on one warp.
#ifndef RTG_COL_CHUNK
#define RTG_COL_CHUNK 10
#endif
constexpr int kColChunk = RTG_COL_CHUNK;
static_assert(kColChunk >= 1 && kColChunk <= 32, "k_col_culled holds one waypoint of a chunk per lane");

template <int kChunk>
__global__ void __launch_bounds__(kWarps * 32) k_col_culled(
    const float* __restrict__ X, const float* __restrict__ Y, const float* __restrict__ Zw, int K, int T,
    const CRec* __restrict__ crec, const CMat* __restrict__ cmat, const CSrc* __restrict__ csrc, const rtg_robot rb,
    const int* __restrict__ cstart, ColGridK g, float gq, int* __restrict__ first_col,
    unsigned char* __restrict__ wp_col, int all_waypoints, int* __restrict__ counter,
    unsigned long long* __restrict__ stats) {
    static_assert(kChunk >= 1 && kChunk <= 32, "k_col_culled holds one waypoint of a chunk per lane");
    const int lane = threadIdx.x & 31;
    const int nch = (T + kChunk - 1) / kChunk;
    const long long items = (long long)K * nch;
    unsigned nref = 0;
    unsigned long long ntest = 0;
    for (;;) {
        int e = 0, fc = 0;
        if (lane == 0) e = atomicAdd(counter, 1);
        e = __shfl_sync(kFull, e, 0);
        if (e >= items) break;
        const int c = e / K, k = e - c * K;
        const int t0 = c * kChunk, t1 = min(T, t0 + kChunk);
        if (lane == 0) fc = *(volatile int*)(first_col + k);
        fc = __shfl_sync(kFull, fc, 0);
        if (!all_waypoints && fc < t0) continue;
        // the chunk's waypoints tested together (lane j holds waypoint t0 + j)
        const long long i0 = (long long)k * T + t0;
        const int nj = t1 - t0;
        float px = NAN, py = NAN, pz = NAN;
        if (lane < nj) {
            px = X[i0 + lane];
            py = Y[i0 + lane];
            pz = Zw[i0 + lane];
        }
        const unsigned hits = warp_points_collide_mask(px, py, pz, nj, !all_waypoints, crec, cmat, csrc, rb, cstart, g,
                                                       gq, nref, ntest);
        if (all_waypoints && lane < nj) wp_col[i0 + lane] = (hits >> lane) & 1u;
        if (hits && lane == 0) atomicMin(first_col + k, t0 + __ffs(hits) - 1);
    }
    if (stats) {
        nref = __reduce_add_sync(kFull, nref);
        if (lane == 0) {
            if (nref) atomicAdd(&stats[0], (unsigned long long)nref);
            atomicAdd(&stats[4], ntest);
        }
    }
}

// ===================================================================== info-waypoint list
// list = { k*T + t : trajectory k computed, (t+1) % stride == 0 }: the computed trajectories ranked by one
// warp-aggregated atomic per warp (k ascending within each warp's 32; the warps' order is the order they
// ran -- the list order only schedules work, every output is indexed by waypoint), each expanded to its
// info waypoints by k_fill_list
__global__ void k_build_list(const int* __restrict__ first_col, int K, int T, int full_gain,
                             int* __restrict__ list, int* __restrict__ nranked) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const bool inc = k < K && (full_gain || first_col[k] == T);
    const unsigned b = __ballot_sync(kFull, inc);
    if (!b) return;
    int base = 0;
    if (lane == 0) base = atomicAdd(nranked, __popc(b));
    base = __shfl_sync(kFull, base, 0);
    if (inc) list[base + __popc(b & ((1u << lane) - 1u))] = k;
}

// list[e] = ranked[e / per] * T + (e % per + 1) * stride - 1 for e < count = ranked count * per (written
// here for the gain kernels)
__global__ void k_fill_list(const int* __restrict__ ranked, const int* __restrict__ nranked, int per, int T,
                            int stride, int* __restrict__ list, int* __restrict__ count) {
    const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long n = (long long)*nranked * per;
    if (e == 0) *count = (int)n;
    if (e >= n) return;
    const int r = (int)(e / per), j = (int)(e - (long long)r * per);
    list[e] = ranked[r] * T + (j + 1) * stride - 1;
}

// identity list (debug: every waypoint)
__global__ void k_iota(int* __restrict__ list, long long n, int* __restrict__ count) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < n) list[i] = (int)i;
    if (i == 0) *count = (int)n;
}

// ===================================================================== dense phase B
constexpr int kDenseGainThreads = 256;
#ifndef RTG_DENSE_GAIN_WPT
#define RTG_DENSE_GAIN_WPT 4
#endif
constexpr int kDenseGainWpt = RTG_DENSE_GAIN_WPT;

__global__ void __launch_bounds__(kDenseGainThreads) k_gain_dense(
    const float* __restrict__ X, const float* __restrict__ Y, const float* __restrict__ Zw,
    const float* __restrict__ Yaw, const int* __restrict__ list, int list_n, const GRec* __restrict__ grec,
    long long n_gain_pad, int tiles_per_split, CamK cam,
    unsigned long long* __restrict__ wp_gq, int* __restrict__ wp_nh, int* __restrict__ wp_nl,
    unsigned long long* __restrict__ stats) {
    __shared__ __align__(128) GRec s_rec[2][kTile];
    __shared__ __align__(8) uint64_t s_bar[2];
    const long long tile0 = (long long)blockIdx.y * tiles_per_split;
    long long ntiles = n_gain_pad / kTile - tile0;
    if (ntiles > tiles_per_split) ntiles = tiles_per_split;
    if (ntiles <= 0) return;

    WpF wf[kDenseGainWpt];
    int wid[kDenseGainWpt];
    bool act[kDenseGainWpt];
    double accq[kDenseGainWpt];   // exact: integers below 2^53
    int nh[kDenseGainWpt], nl[kDenseGainWpt];
#pragma unroll
    for (int j = 0; j < kDenseGainWpt; ++j) {
        int e = blockIdx.x * (kDenseGainThreads * kDenseGainWpt) + j * kDenseGainThreads + threadIdx.x;
        act[j] = e < list_n;
        int i = act[j] ? list[e] : list[0];
        wid[j] = i;
        float x = X[i], y = Y[i], z = Zw[i], yw = Yaw[i];
        act[j] = act[j] && isfinite(x) && isfinite(y) && isfinite(z) && isfinite(yw);
        if (!act[j]) { x = __int_as_float(0x7fc00000); y = x; z = x; yw = 0.f; }   // NaN pose: sees nothing
        wp_setup(x, y, z, yw, cam, wf[j]);
        accq[j] = 0.0;
        nh[j] = 0;
        nl[j] = 0;
    }
    static_assert(kDenseGainWpt % 2 == 0, "waypoints go in pairs (packed FP32)");
    WpF2 wp2[kDenseGainWpt / 2];
#pragma unroll
    for (int j = 0; j < kDenseGainWpt; j += 2) wp2[j / 2] = wp_pair(wf[j], wf[j + 1]);
    if (threadIdx.x == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const uint32_t rb = kTile * sizeof(GRec);
    if (threadIdx.x == 0) {
        for (int s = 0; s < 2 && s < ntiles; ++s) {
            mbar_expect_tx(&s_bar[s], rb);
            bulk_g2s(s_rec[s], grec + (tile0 + s) * kTile, rb, &s_bar[s]);
        }
    }
    unsigned nref = 0;
    for (long long it = 0; it < ntiles; ++it) {
        const int s = (int)(it & 1);
        mbar_wait(&s_bar[s], (uint32_t)((it >> 1) & 1));
        const GRec* rec = s_rec[s];
        // exact integer sums per half tile: 256 u_q < 2^24 fit 32 bits, 512 class increments the
        // packed nH | nL << 16 counter
        int pc[kDenseGainWpt];
#pragma unroll
        for (int j = 0; j < kDenseGainWpt; ++j) pc[j] = 0;
        for (int h = 0; h < kTile; h += kTile / 2) {
            unsigned qs[kDenseGainWpt];
#pragma unroll
            for (int j = 0; j < kDenseGainWpt; ++j) qs[j] = 0;
#pragma unroll 2
            for (int g = h; g < h + kTile / 2; ++g) {
                const GRec G = rec[g];
                const unsigned q = G.uc & kUqMask;
                const int inc = uc_inc(G.uc);
                float m[kDenseGainWpt], gd[kDenseGainWpt];
#pragma unroll
                for (int j = 0; j < kDenseGainWpt; j += 2)
                    vis_margin_w2(wp2[j / 2], cam, G.x, G.y, G.z, m[j], m[j + 1], gd[j], gd[j + 1]);
                bool v[kDenseGainWpt], amb = false;
#pragma unroll
                for (int j = 0; j < kDenseGainWpt; ++j) {
                    v[j] = m[j] >= 0.0f;
                    amb |= fabsf(m[j]) < gd[j];
                }
                if (amb) {   // FP32 guard band: FP64 re-decision (rare)
#pragma unroll
                    for (int j = 0; j < kDenseGainWpt; ++j) {
                        if (fabsf(m[j]) < gd[j]) {
                            v[j] = vis_decide64(wf[j].px, wf[j].py, wf[j].pz, wf[j].yaw, G.x, G.y, G.z, cam.cam64);
                            ++nref;
                        }
                    }
                }
#pragma unroll
                for (int j = 0; j < kDenseGainWpt; ++j) {
                    if (v[j]) {
                        qs[j] += q;
                        pc[j] += inc;
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < kDenseGainWpt; ++j) accq[j] += (double)qs[j];
        }
#pragma unroll
        for (int j = 0; j < kDenseGainWpt; ++j) {
            nh[j] += pc[j] & 0xffff;
            nl[j] += pc[j] >> 16;
        }
        __syncthreads();
        if (threadIdx.x == 0 && it + 2 < ntiles) {
            mbar_expect_tx(&s_bar[s], rb);
            bulk_g2s(s_rec[s], grec + (tile0 + it + 2) * kTile, rb, &s_bar[s]);
        }
    }
#pragma unroll
    for (int j = 0; j < kDenseGainWpt; ++j) {
        if (act[j]) {
            if (accq[j] != 0.0) atomicAdd(&wp_gq[wid[j]], (unsigned long long)(long long)accq[j]);
            if (nh[j]) atomicAdd(&wp_nh[wid[j]], nh[j]);
            if (nl[j]) atomicAdd(&wp_nl[wid[j]], nl[j]);
        }
    }
    if (stats && nref) atomicAdd(&stats[1], (unsigned long long)nref);
}

// ===================================================================== a6 reduction
__global__ void k_reduce(int K, int T, int stride, int variant, float lambda_xi, int full_gain,
                         const int* __restrict__ first_col, const long long* __restrict__ wp_gq,
                         const int* __restrict__ wp_nh, const int* __restrict__ wp_nl,
                         const StartState* __restrict__ start,
                         const ClassState* __restrict__ cs, int* __restrict__ out_first,
                         unsigned char* __restrict__ out_feasible, double* __restrict__ out_gain,
                         double* __restrict__ out_util) {
    const int lane = threadIdx.x & 31;
    const int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (k >= K) return;
    const int fc = first_col[k];
    const bool feasible = fc >= T;
    const bool computed = feasible || full_gain;
    long long q = 0, h = 0, l = 0;
    if (computed) {
        if (start && lane == 0) {   // info state l = 0, the shared start (Eq. equ:traj_utility)
            q = start->gq;
            h = start->nh;
            l = start->nl;
        }
        for (int t = stride - 1 + lane * stride; t < T; t += 32 * stride) {
            long long i = (long long)k * T + t;
            q += wp_gq[i];
            h += wp_nh[i];
            l += wp_nl[i];
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        q += __shfl_xor_sync(kFull, q, o);
        h += __shfl_xor_sync(kFull, h, o);
        l += __shfl_xor_sync(kFull, l, o);
    }
    if (lane == 0) {
        const double nan = __longlong_as_double(0x7ff8000000000000LL);
        double gain = computed ? (double)q * cs->inv_scale : nan;
        double xi = (double)h - (double)lambda_xi * (double)l;
        double util = feasible ? (variant == RTG_VARIANT_SUM ? gain : xi) : -INFINITY;
        if (out_first) out_first[k] = feasible ? T : fc;
        if (out_feasible) out_feasible[k] = feasible ? 1 : 0;
        if (out_gain) out_gain[k] = gain;
        if (out_util) out_util[k] = util;
    }
}

// per-waypoint debug outputs
__global__ void k_debug_wp(long long n, const long long* __restrict__ wp_gq, const ClassState* __restrict__ cs,
                           double* __restrict__ out_gain) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < n) out_gain[i] = (double)wp_gq[i] * cs->inv_scale;
}

// ===================================================================== a7 argmax
struct BestDev {
    double score;
    long long index;
};

__global__ void k_best(const double* __restrict__ u, int K, long long base, BestDev* __restrict__ out) {
    __shared__ double sv[1024];
    __shared__ int si[1024];
    double bv = -INFINITY;
    int bi = -1;
    // eight loads in flight per thread (a single block reads all K: one dependent load per step would
    // cost K / blockDim.x memory latencies), then compared in index order
    constexpr int kU = 8;
    for (int k0 = threadIdx.x; k0 < K; k0 += kU * blockDim.x) {
        double v[kU];
#pragma unroll
        for (int j = 0; j < kU; ++j) {
            const int k = k0 + j * (int)blockDim.x;
            v[j] = k < K ? u[k] : -INFINITY;
        }
#pragma unroll
        for (int j = 0; j < kU; ++j) {
            if (v[j] > bv) {   // strict: keeps the lowest index among equal values (k ascending per thread)
                bv = v[j];
                bi = k0 + j * (int)blockDim.x;
            }
        }
    }
    sv[threadIdx.x] = bv;
    si[threadIdx.x] = bi;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) {
            double ov = sv[threadIdx.x + s];
            int oi = si[threadIdx.x + s];
            double mv = sv[threadIdx.x];
            int mi = si[threadIdx.x];
            if (oi >= 0 && (mi < 0 || ov > mv || (ov == mv && oi < mi))) {
                sv[threadIdx.x] = ov;
                si[threadIdx.x] = oi;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out->score = si[0] >= 0 ? sv[0] : -INFINITY;
        out->index = si[0] >= 0 ? base + si[0] : -1;
    }
}

// ===================================================================== debug pair mask
__global__ void k_pair_mask(const float* __restrict__ X, const float* __restrict__ Y, const float* __restrict__ Zw,
                            long long KT, long long N, const CRec* __restrict__ crec, const CMat* __restrict__ cmat,
                            const CSrc* __restrict__ csrc, const rtg_robot rb, long long n_col, float gq,
                            unsigned int* __restrict__ mask) {
    long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (idx >= KT * n_col) return;
    long long i = idx / n_col, g = idx % n_col;
    float px = X[i], py = Y[i], pz = Zw[i];
    const CRec A = crec[g];
    float dx = px - A.x, dy = py - A.y, dz = pz - A.z;
    float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
    unsigned nref = 0;
    if (d2 < A.rb2 &&
        collide_full(cmat[g].m, dx, dy, dz, gq, &csrc[g], rb, px, py, pz, A.x, A.y, A.z, nref)) {
        long long orig = __float_as_int(cmat[g].m[9]);
        unsigned long long bit = (unsigned long long)(i * N + orig);
        atomicOr(&mask[bit >> 5], 1u << (bit & 31));
    }
}

// ===================================================================== sampler (a3)
__global__ void k_sample_unicycle(int K, int T, double dt, double x0, double y0, double z0, double th0,
                                  const float* __restrict__ v, const float* __restrict__ om, float* __restrict__ X,
                                  float* __restrict__ Y, float* __restrict__ Zw, float* __restrict__ Yaw) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= (long long)K * T) return;
    int k = (int)(i / T), l = (int)(i % T);
    double vv = v[k], ww = om[k];
    double t = (l + 1) * dt;
    double th = th0 + ww * t;
    double x, y;
    if (fabs(ww) < 1e-12) {
        x = x0 + vv * t * cos(th0);
        y = y0 + vv * t * sin(th0);
    } else {
        x = x0 + (vv / ww) * (sin(th) - sin(th0));
        y = y0 + (vv / ww) * (cos(th0) - cos(th));
    }
    double wr = remainder(th, 2.0 * M_PI);   // in [-pi, pi]
    if (wr <= -M_PI) wr += 2.0 * M_PI;
    X[i] = (float)x;
    Y[i] = (float)y;
    Zw[i] = (float)z0;
    Yaw[i] = (float)wr;
}

// double-integrator primitives (BASELINE.json configs[2]): constant acceleration (ax, ay)[k] from
// (x0, y0) with velocity (vx, vy); t_l = (l+1) dt; heading along the velocity; FP64, stored as FP32
__global__ void k_sample_double_integrator(int K, int T, double dt, double x0, double y0, double z0, double vx,
                                           double vy, const float* __restrict__ ax, const float* __restrict__ ay,
                                           float* __restrict__ X, float* __restrict__ Y, float* __restrict__ Zw,
                                           float* __restrict__ Yaw) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= (long long)K * T) return;
    const int k = (int)(i / T), l = (int)(i % T);
    const double a = ax[k], b = ay[k];
    const double t = __dmul_rn((double)(l + 1), dt);
    const double t2 = __dmul_rn(t, t);
    X[i] = (float)__dadd_rn(__dadd_rn(x0, __dmul_rn(vx, t)), __dmul_rn(__dmul_rn(0.5, a), t2));
    Y[i] = (float)__dadd_rn(__dadd_rn(y0, __dmul_rn(vy, t)), __dmul_rn(__dmul_rn(0.5, b), t2));
    Zw[i] = (float)z0;
    Yaw[i] = (float)atan2(__dadd_rn(vy, __dmul_rn(b, t)), __dadd_rn(vx, __dmul_rn(a, t)));
}

// ===================================================================== host launchers
cudaError_t launch_gain_culled(rtg_map_s* m, rtg_traj_s* tr, const CamK& cam, const int* list, const int* count,
                               long long list_max, long long* wp_gq, int* wp_nh, int* wp_nl, int* counter,
                               unsigned long long* stats, cudaStream_t st);
namespace {
int g_occ_col = 0, g_sms = 0;
void occupancy(int dev) {
    if (g_sms) return;
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_occ_col, k_col_culled<kColChunk>, kWarps * 32, 0);
    if (g_occ_col < 1) g_occ_col = 1;
}
}  // namespace

CamK make_cam(const rtg_camera& c, const double* cam64_dev) {
    CamK k;
    double W = c.width, H = c.height, fx = c.fx, fy = c.fy, cx = c.cx, cy = c.cy, zn = c.z_near, zf = c.z_far;
    double kxl = cx / fx, kxr = (W - cx) / fx, kyu = cy / fy, kyd = (H - cy) / fy;
    k.zmid = (float)(0.5 * (zn + zf));
    k.zhalf = (float)(0.5 * (zf - zn));
    k.kxc = (float)(0.5 * (kxr - kxl));
    k.kxh = (float)(0.5 * (kxr + kxl));
    k.kyc = (float)(0.5 * (kyu - kyd));
    k.kyh = (float)(0.5 * (kyu + kyd));
    // FP32 error bound of the min slack, doubled
    const double u = ldexp(1.0, -24);
    double kxm = fabs(k.kxc) + k.kxh, kym = fabs(k.kyc) + k.kyh;
    k.gam = (float)(24.0 * u * (1.0 + kxm) * (1.0 + kym) * sqrt(1.0 + kxm * kxm) * 2.0);
    k.g0 = (float)(8.0 * u * (fabs(k.zmid) + k.zhalf + 1.0));
    k.cam64 = cam64_dev;
    return k;
}

cudaError_t launch_phase_a(rtg_map_s* m, rtg_traj_s* tr, int mode, int* first_col, unsigned char* wp_col,
                           int all_wp, int* counter, unsigned long long* stats, cudaStream_t st) {
    occupancy(m->device);
    const int K = tr->K, T = tr->T;
    if (mode == RTG_MODE_DENSE) {
        long long KT = (long long)K * T;
        int wblocks = (int)((KT + kDenseColThreads * kDenseColWpt - 1) / (kDenseColThreads * kDenseColWpt));
        long long ntiles = m->n_col_pad / kTile;
        if (ntiles == 0) return cudaGetLastError();
        long long want = (long long)g_sms * 8;
        long long splits = (want + wblocks - 1) / wblocks;
        if (splits > ntiles) splits = ntiles;
        if (splits < 1) splits = 1;
        int tps = (int)((ntiles + splits - 1) / splits);
        splits = (ntiles + tps - 1) / tps;
        dim3 grid(wblocks, (unsigned)splits);
        note_launch(), k_col_dense<<<grid, kDenseColThreads, 0, st>>>(tr->x, tr->y, tr->z, K, T, m->crec, m->cmat, m->csrc, m->robot,
                                                       m->n_col_pad, tps, m->gq, first_col, wp_col, all_wp, stats);
    } else {
        if (m->n_col == 0) return cudaGetLastError();
        ColGridK g;
        g.ox = m->cg.ox; g.oy = m->cg.oy; g.oz = m->cg.oz; g.h = m->cg.h;
        g.R = m->rb_max * (1.0f + 2e-5f) + 1e-4f;
        g.nx = m->cg.nx; g.ny = m->cg.ny; g.nz = m->cg.nz;
        // waypoints per work item: kColChunk (10), or 5 / 3 when that would leave fewer than 20 work items per
        // resident warp (small plans: the kernel is latency-bound, so the chunks' parallelism beats the shared
        // candidate loads; measured: room 0.140 -> 0.069 ms at 3, multi-room 0.134 -> 0.090 at 5,
        // outdoor and scale stay at 10)
        const long long slots = (long long)g_sms * g_occ_col * kWarps;
        int chunk = 3;
        for (const int c : {kColChunk, 5}) {
            if (c <= kColChunk && (long long)K * ((T + c - 1) / c) >= 20 * slots) {
                chunk = c;
                break;
            }
        }
        if (chunk > kColChunk) chunk = kColChunk;
        const char* chunk_var = getenv("RTG_COL_CHUNK_RT");   // (read per call: the parity test switches it)
        const int chunk_env = chunk_var ? atoi(chunk_var) : 0;
        if (chunk_env == 3 || chunk_env == 5 || chunk_env == kColChunk) chunk = chunk_env;   // (A/B measurements)
        const long long items = (long long)K * ((T + chunk - 1) / chunk);
        int blocks = (int)std::min<long long>((items + kWarps - 1) / kWarps, 1LL << 30);
        int cap = g_sms * g_occ_col;
        if (blocks > cap) blocks = cap;
#define RTG_COL_LAUNCH(C)                                                                                         \
    note_launch(), k_col_culled<C><<<blocks, kWarps * 32, 0, st>>>(tr->x, tr->y, tr->z, K, T, m->crec, m->cmat,       \
                                                                   m->csrc, m->robot, m->cstart, g, m->gq, first_col, \
                                                                   wp_col, all_wp, counter, stats)
        if (chunk == 3) RTG_COL_LAUNCH(3);
        else if (chunk == 5) RTG_COL_LAUNCH(5);
        else RTG_COL_LAUNCH(kColChunk);
#undef RTG_COL_LAUNCH
    }
    return cudaGetLastError();
}

cudaError_t launch_list(const int* first_col, int K, int T, int stride, int full_gain, int* list, int* count,
                        int* ranked, cudaStream_t st) {
    // count[4]: the ranked trajectories (zeroed with the scratch; count[1], count[2] are the collision and
    // gain kernels' work counters), count[0]: the list length
    note_launch(), k_build_list<<<(unsigned)((K + 255) / 256), 256, 0, st>>>(first_col, K, T, full_gain, ranked,
                                                                             count + 4);
    const long long per = T / stride, n = (long long)K * per;
    note_launch(), k_fill_list<<<(unsigned)(n > 0 ? (n + 255) / 256 : 1), 256, 0, st>>>(ranked, count + 4, (int)per,
                                                                                       T, stride, list, count);
    return cudaGetLastError();
}

cudaError_t launch_iota(int* list, long long n, int* count, cudaStream_t st) {
    note_launch(), k_iota<<<(unsigned)((n + 255) / 256 > 0 ? (n + 255) / 256 : 1), 256, 0, st>>>(list, n, count);
    return cudaGetLastError();
}

// dense phase B needs the list length on the host (one sync; dense mode is the brute-force path)
cudaError_t launch_phase_b(rtg_map_s* m, rtg_traj_s* tr, int mode, const CamK& cam, const int* list,
                           const int* count, long long list_max, long long* wp_gq, int* wp_nh, int* wp_nl,
                           int* counter, unsigned long long* stats, cudaStream_t st) {
    occupancy(m->device);
    if (mode == RTG_MODE_DENSE) {
        int n = 0;
        cudaError_t e = cudaMemcpyAsync(&n, count, sizeof(int), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return e;
        long long ntiles = m->n_gain_pad / kTile;
        if (n == 0 || ntiles == 0) return cudaGetLastError();
        int per_block = kDenseGainThreads * kDenseGainWpt;
        int wblocks = (n + per_block - 1) / per_block;
        long long want = (long long)g_sms * 8;
        long long splits = (want + wblocks - 1) / wblocks;
        if (splits > ntiles) splits = ntiles;
        if (splits < 1) splits = 1;
        int tps = (int)((ntiles + splits - 1) / splits);
        splits = (ntiles + tps - 1) / tps;
        dim3 grid(wblocks, (unsigned)splits);
        note_launch(), k_gain_dense<<<grid, kDenseGainThreads, 0, st>>>(tr->x, tr->y, tr->z, tr->yaw, list, n, m->grec,
                                                         m->n_gain_pad, tps, cam, (unsigned long long*)wp_gq, wp_nh,
                                                         wp_nl, stats);
    } else {
        return launch_gain_culled(m, tr, cam, list, count, list_max, wp_gq, wp_nh, wp_nl, counter, stats, st);
    }
    return cudaGetLastError();
}

__global__ void k_start_setup(float x, float y, float z, float yaw, StartState* __restrict__ s) {
    if (threadIdx.x == 0) {
        s->pose[0] = x;
        s->pose[1] = y;
        s->pose[2] = z;
        s->pose[3] = yaw;
        s->gq = 0;
        s->nh = 0;
        s->nl = 0;
        s->list[0] = 0;
        s->count[0] = 1;
        s->counter[0] = 0;
    }
}

cudaError_t launch_start_setup(const float pose[4], StartState* s, cudaStream_t st) {
    note_launch(), k_start_setup<<<1, 32, 0, st>>>(pose[0], pose[1], pose[2], pose[3], s);
    return cudaGetLastError();
}

cudaError_t launch_reduce(rtg_map_s* m, rtg_traj_s* tr, const rtg_score_params& p, const int* first_col,
                          const long long* wp_gq, const int* wp_nh, const int* wp_nl, const StartState* start,
                          int* out_first, unsigned char* out_feasible, double* out_gain, double* out_util,
                          cudaStream_t st) {
    int K = tr->K;
    int threads = 256;
    int blocks = (int)(((long long)K * 32 + threads - 1) / threads);
    note_launch(), k_reduce<<<blocks, threads, 0, st>>>(K, tr->T, p.info_stride, p.variant, p.lambda_xi,
                                         (p.flags & RTG_SCORE_FULL_GAIN) ? 1 : 0, first_col, wp_gq, wp_nh, wp_nl,
                                         start, m->cls, out_first, out_feasible, out_gain, out_util);
    return cudaGetLastError();
}

cudaError_t launch_debug_wp(long long n, const long long* wp_gq, const ClassState* cs, double* out, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    note_launch(), k_debug_wp<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, wp_gq, cs, out);
    return cudaGetLastError();
}

cudaError_t launch_pair_mask(rtg_map_s* m, rtg_traj_s* tr, unsigned* mask, cudaStream_t st) {
    long long KT = (long long)tr->K * tr->T;
    long long tot = KT * m->n_col;
    if (tot == 0) return cudaSuccess;
    note_launch(), k_pair_mask<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(tr->x, tr->y, tr->z, KT, m->n, m->crec, m->cmat,
                                                                m->csrc, m->robot, m->n_col, m->gq, mask);
    return cudaGetLastError();
}

// the FP64 camera for the re-decision branch, written by a kernel (its values travel as launch
// parameters, so rtg_score stays capturable in a CUDA graph: no pageable host copy)
struct Cam64Args { double v[8]; };
__global__ void k_set_cam64(Cam64Args a, double* __restrict__ dst) {
    if (threadIdx.x < 8) dst[threadIdx.x] = a.v[threadIdx.x];
}

cudaError_t launch_set_cam64(const rtg_camera& c, double* dst, cudaStream_t st) {
    const Cam64Args a{{(double)c.width, (double)c.height, c.fx, c.fy, c.cx, c.cy, c.z_near, c.z_far}};
    note_launch(), k_set_cam64<<<1, 32, 0, st>>>(a, dst);
    return cudaGetLastError();
}

cudaError_t launch_best(const double* u, int K, long long base, void* out_dev, cudaStream_t st) {
    note_launch(), k_best<<<1, 1024, 0, st>>>(u, K, base, (BestDev*)out_dev);
    return cudaGetLastError();
}

cudaError_t launch_sampler_di(int K, int T, double dt, const float* start, const float* v0, const float* ax,
                              const float* ay, rtg_traj_s* tr, cudaStream_t st) {
    const long long n = (long long)K * T;
    note_launch(), k_sample_double_integrator<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
                       K, T, dt, start[0], start[1], start[2], v0[0], v0[1], ax, ay, tr->x, tr->y, tr->z, tr->yaw);
    return cudaGetLastError();
}

cudaError_t launch_sampler(int K, int T, double dt, const float* start, const float* v, const float* om,
                           rtg_traj_s* tr, cudaStream_t st) {
    long long n = (long long)K * T;
    note_launch(), k_sample_unicycle<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(K, T, dt, start[0], start[1], start[2], start[3],
                                                                   v, om, tr->x, tr->y, tr->z, tr->yaw);
    return cudaGetLastError();
}

}  // namespace rtg
