// rtg_gain_culled.cu -- exact culled visibility + information gain.
//
// One warp per info waypoint (persistent warps, 4-warp CTAs x 9 per SM at 56 registers, pull
// waypoints from an atomic counter in (k, t) order).  The frustum is six linear constraints
// f_j(p) = a_j dx + b_j dy + g_j dz + d_j >= 0 (the pinhole slacks of O3: near, far, two side planes
// through the camera centre, top and bottom); over a grid cell (box) the minimum / maximum of each is
// its centre value -/+ a radius, and along a grid row the centre value is linear in the x-cell
// index, so the cells of a row that are possibly visible / fully inside form index intervals found
// with one multiply per constraint.  Per waypoint:
//   1. lanes take the grid rows (y bands) the frustum's footprint covers, 32 at a time; per row the
//      four horizontal constraints give the x-interval P of possibly visible columns and its
//      sub-interval I of columns whose whole column box is horizontally inside;
//   2. the flanks P \ I are tested Gaussian by Gaussian from record copy A (sorted by
//      (row, x-cell, z-cell)): each flank is ONE contiguous record run (all z);
//   3. the inside columns I are walked z-cell by z-cell from copy B (sorted by (row, z-cell,
//      x-cell), so a row's z-slab is x-contiguous): per (row, z-cell) unit (lanes flattened over the
//      chunk's units through a shared-memory owner table) the two vertical constraints cut I into an
//      x-run fully inside (added from the exact prefixes of the z-fastest table: the difference of
//      two 16-byte entries {start, prefixes mod 2^48 / 2^24}) and at most two straddling x-runs
//      (tested); the z-cells a row can see come from the vertical wedge at the row's largest depth
//      and the row's occupied z-range;
//   4. tested runs go to a per-warp queue; a flush tests 64 items per pass, two per lane, whatever
//      the run lengths: a shared-memory bitmap marks the items where runs start (shifted by one), so
//      each lane finds its run from a 64-bit window of it (one broadcast load, popc); items past the
//      queue fall in a sentinel run of NaN padding records (never visible, so no bound check).
//      The pair test is the shared exact one (packed FP32 + FP64 re-decision inside the proven
//      guard band).
// Sums are exact integers (24-bit u_q and a class byte per record, 32-bit per-lane sums flushed
// into 64-bit ones; integer prefixes): order free, so the result is bit-identical to the dense
// kernel.  eps (>> FP32 error of the cell tests) keeps "inside" strictly inside and "possible" a
// superset.
#include <cfloat>
#include <climits>
#include <cstdio>
#include <cstdlib>

#include "rtg_host.hpp"

namespace rtg {
namespace {

constexpr unsigned kFullG = 0xffffffffu;
constexpr int kWarpsG = 4;     // warps per CTA; RTG_GAIN_MINB CTAs per SM: 36 warps at 56 registers
constexpr int kQCap = 256;    // queued runs per warp
#ifndef RTG_QFLUSH
#define RTG_QFLUSH 192
#endif
constexpr int kQFlush = RTG_QFLUSH;  // test the queue once more runs than this are waiting (an append adds <= 64)
static_assert(kQFlush + 64 <= kQCap, "the flush prefix takes 8 runs per lane: at most 256 queued runs");
constexpr int kMaxUnits = 1024;   // units of a row chunk with a shared-memory owner table (else: search)
constexpr int kHeadWords = (64 * 63 + 64 + 32) / 32 + 1;   // a flush chunk (kFlushPasses passes) + the window tail

// RTG_BOUNDS_CHECK builds trap on any out-of-range table or record index (debug builds; the
// sanitizer is not available on the GPU pool)
#ifdef RTG_BOUNDS_CHECK
#define RTG_CHECK(cond, what)                                                                     \
    do {                                                                                          \
        if (!(cond)) {                                                                            \
            printf("rtg bounds: %s (block %d thread %d)\n", what, (int)blockIdx.x, (int)threadIdx.x); \
            __trap();                                                                             \
        }                                                                                         \
    } while (0)
#else
#define RTG_CHECK(cond, what) ((void)0)
#endif

struct GainK {
    float ox, oy, oz, hx, hy, hz, inv_hz, eps;
    int nx, ny, nz, nxb, offB;
    long long nrec, ntabB, ntabA;   // sizes (bounds checks)
    int nan_rec;                    // first of >= 64 NaN padding records (copy A's tail): sentinel run
    float zn, zf, kxl, kxr, kyu, kyd, kxh;
};

// 9 x 4 warps: 56 registers without spills (measured: 32 warps / 64 registers 4.7 % slower, 40 warps /
// 48 registers spill and are 16 % slower, 28 warps / 72 registers 6 % slower)
#ifndef RTG_GAIN_MINB
#define RTG_GAIN_MINB 9
#endif

__device__ __forceinline__ int fcell(float v, int hi) {   // floor of v clamped to [-1, hi + 1]
    v = fminf(fmaxf(v, -1.0f), (float)hi + 1.0f);
    return (int)floorf(v);
}

// constraint j seen by grid cell (ix, iy, iz): centre value = A ix + B iy + G iz + K, box radius r;
// stored as {K, B, inv = 1/A, e = eps + r} (G = 0 for the horizontal ones, -+hz for top / bottom).
// cut() tightens [plo, phi] (possibly visible: A ix >= -e - Cj) and [ilo, ihi] (inside:
// A ix >= e - Cj) with Cj the centre value at ix = 0.
__device__ __forceinline__ void cut(const float4& C, float Cj, float& plo, float& phi, float& ilo, float& ihi) {
    const float tp = (-C.w - Cj) * C.z, ti = (C.w - Cj) * C.z;
    if (C.z > 0.f) {
        plo = fmaxf(plo, ceilf(tp));
        ilo = fmaxf(ilo, ceilf(ti));
    } else {
        phi = fminf(phi, floorf(tp));
        ihi = fminf(ihi, floorf(ti));
    }
}

// w += uc and pc += class byte of record word uc when p: over at most kFlushPasses passes (2 items
// each) w - (pc << 24) = sum(u_q) < 2^32 and pc = nH + 128 nL with nH <= 126 (both exact)
constexpr int kFlushPasses = 63;
__device__ __forceinline__ void add_if(bool p, unsigned& w, unsigned uc, unsigned& pc) {
    if (p) {
        w += uc;
        pc += __byte_perm(uc, 0u, 0x4443);   // the class byte (top byte of uc)
    }
}

template <bool kStats, bool kLongRuns>
__global__ void __launch_bounds__(kWarpsG * 32, RTG_GAIN_MINB) k_gain_culled(
    const float* __restrict__ X, const float* __restrict__ Y, const float* __restrict__ Zw,
    const float* __restrict__ Yaw, const int* __restrict__ list, const int* __restrict__ list_count,
    const double2* __restrict__ trig, const GRec* __restrict__ grec, const int* __restrict__ gstartA,
    const int2* __restrict__ zocc, const TabP* __restrict__ gtabP, const GainK g,
    const CamK cam, long long* __restrict__ wp_gq, int* __restrict__ wp_nh, int* __restrict__ wp_nl,
    int* __restrict__ counter, unsigned long long* __restrict__ stats) {
    // per-warp state, one struct per warp so a single base register addresses all of it
    struct __align__(16) WarpSmem {
        float4 con[6];                       // the frustum's constraints on grid cells
        double cs[2];                        // FP64 cos, sin of the waypoint's yaw (re-decisions)
        float v[8];                          // footprint vertices (x0..x3, y0..y3), grid-relative
        // queued test runs: [0] first record -> (first record - items before the run), [1] length;
        // entry nq of [0] is the sentinel run (NaN records) while the queue is tested
        int q[2][kQCap + 64];
        unsigned head[kHeadWords];           // run-start bitmap of the flush chunk being tested
        unsigned char owner[kMaxUnits];      // row (lane) of each unit of the current chunk
    };
    __shared__ WarpSmem s_w[kWarpsG];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned lanes_lt;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lanes_lt));
    WarpSmem& sw = s_w[wid];
    int* const qs = sw.q[0];
    int* const qe = sw.q[1];
    for (int j = lane; j < kHeadWords; j += 32) sw.head[j] = 0u;   // kept all-zero between flush chunks
    __syncwarp();
    const int L = *list_count;
    unsigned nref = 0;
    unsigned long long ntest = 0, nagg = 0, nunit = 0, nflank = 0, nvis = 0, nrow = 0, nruns = 0, ntab = 0, nrowb = 0;
    for (;;) {
        int e = 0;
        if (lane == 0) e = atomicAdd(counter, 1);
        e = __shfl_sync(kFullG, e, 0);
        if (e >= L) break;
        const int i = list[e];
        const float px = X[i], py = Y[i], pz = Zw[i], yw = Yaw[i];
        unsigned long long acc = 0;  // sum of u_q over visible Gaussians (exact integer)
        int acch = 0, accl = 0;
        if (isfinite(px) && isfinite(py) && isfinite(pz) && isfinite(yw)) {
            WpF f;
            {
                const double2 t2 = trig[e];   // FP64 (cos, sin) of the yaw, one per list entry (k_wp_trig)
                const double cs = t2.x, sn = t2.y;
                wp_setup_from_cs(px, py, pz, yw, cs, sn, cam, f);
                const float qx = px - g.ox, qy = py - g.oy;
                if (lane < 4) {     // vertex = p + Z (c, s) + kZ (s, -c)
                    const float zz = lane < 2 ? g.zn : g.zf;
                    const float kk = (lane == 0 || lane == 3) ? -g.kxl : g.kxr;
                    sw.v[lane] = fmaf(zz, fmaf(kk, f.s, f.c), qx);
                    sw.v[4 + lane] = fmaf(zz, fmaf(-kk, f.c, f.s), qy);
                }
                if (lane < 6) {
                    // Z = c dx + s dy, X' = ax dx + bx dy (X - kxc Z), constraint j:
                    //   0: Z - zn  1: zf - Z  2: kxh Z - X'  3: kxh Z + X'  4: kyu Z - dz  5: kyd Z + dz
                    float a, b, gz = 0.f, d = 0.f;
                    if (lane == 0) { a = f.c; b = f.s; d = -g.zn; }
                    else if (lane == 1) { a = -f.c; b = -f.s; d = g.zf; }
                    else if (lane == 2) { a = fmaf(g.kxh, f.c, -f.ax); b = fmaf(g.kxh, f.s, -f.bx); }
                    else if (lane == 3) { a = fmaf(g.kxh, f.c, f.ax); b = fmaf(g.kxh, f.s, f.bx); }
                    else if (lane == 4) { a = g.kyu * f.c; b = g.kyu * f.s; gz = -1.f; }
                    else { a = g.kyd * f.c; b = g.kyd * f.s; gz = 1.f; }
                    // cell-centre offsets from the waypoint at index 0
                    const float X0 = fmaf(0.5f, g.hx, -qx), Y0 = fmaf(0.5f, g.hy, -qy);
                    const float Z0 = fmaf(0.5f, g.hz, g.oz - pz);
                    const float A = a * g.hx, B = b * g.hy;
                    sw.con[lane] = make_float4(fmaf(a, X0, fmaf(b, Y0, fmaf(gz, Z0, d))), B,
                                                   fabsf(A) > 1e-30f ? 1.0f / A : 1e30f,
                                                   g.eps + 0.5f * (fabsf(A) + fabsf(B) + fabsf(gz) * g.hz));
                }
                if (lane == 0) {
                    sw.cs[0] = cs;
                    sw.cs[1] = sn;
                }
                __syncwarp();
            }
            const float ymn = fminf(fminf(sw.v[4], sw.v[5]), fminf(sw.v[6], sw.v[7])) - g.eps;
            const float ymx = fmaxf(fmaxf(sw.v[4], sw.v[5]), fmaxf(sw.v[6], sw.v[7])) + g.eps;
            const float inv_hy = 1.0f / g.hy;
            const int iy0 = max(0, fcell(ymn * inv_hy, g.ny));
            const int iy1 = min(g.ny - 1, fcell(ymx * inv_hy, g.ny));
            const float zrel = pz - g.oz;
            // producer / consumer loop: each pass produces one row chunk (32 rows: flank runs) or
            // one window of 32 (row, z-cell) units (aggregates + straddling runs), queues the
            // runs, and tests the queue once it holds more than kQFlush runs (all of it at the end)
            int nq = 0;                      // queued runs (warp-uniform)
            int rnext = iy0, rcur = 0;       // next / current row chunk
            int U = 0, ub = 0;               // units of the current chunk, next unit window
            int incl = 0, zoff = 0, ri0 = 0, ri1 = 0;   // lane's row of the current chunk
            for (;;) {
                int s0 = 0, l0 = 0, s1 = 0, l1 = 0;
                bool done = false;
                if (ub < U) {
                    // ---- unit window: (row, z-cell) units ub .. ub + 31 of the current chunk
                    const int pos = ub + lane;
                    int owner = 0;   // first lane whose inclusive prefix exceeds pos
                    if (U <= kMaxUnits) {
                        owner = pos < U ? sw.owner[pos] : 31;
                    } else {
#pragma unroll
                        for (int st = 16; st > 0; st >>= 1) {
                            const int v = __shfl_sync(kFullG, incl, owner + st - 1);
                            if (v <= pos) owner += st;
                        }
                    }
                    const int iz = pos + __shfl_sync(kFullG, zoff, owner);
                    const int ui0 = __shfl_sync(kFullG, ri0, owner), ui1 = __shfl_sync(kFullG, ri1, owner);
                    const int uy = rcur + owner;
                    const float fuy = (float)uy, fiz = (float)iz;
                    float vplo = (float)ui0, vphi = (float)ui1, vilo = vplo, vihi = vphi;
                    {
                        const float4 Ct = sw.con[4], Cb = sw.con[5];
                        cut(Ct, fmaf(Ct.y, fuy, fmaf(-g.hz, fiz, Ct.x)), vplo, vphi, vilo, vihi);
                        cut(Cb, fmaf(Cb.y, fuy, fmaf(g.hz, fiz, Cb.x)), vplo, vphi, vilo, vihi);
                    }
                    const int q0 = (int)fminf(vplo, (float)g.nx), q1 = pos < U ? (int)vphi : -1;
                    const int j0 = max((int)fminf(vilo, (float)g.nx), q0), j1 = min((int)vihi, q1);
                    if (q0 <= q1) {
                        // z-fastest table: entry (uy, x, iz) at (uy * (nx + 1) + x) * nz + iz
                        // all lookups independent: one memory round trip per unit
                        const int ub0 = uy * (g.nx + 1) * g.nz + iz;
                        const int4* tp = reinterpret_cast<const int4*>(gtabP) + ub0;
                        const bool in = j0 <= j1;
                        RTG_CHECK(uy >= 0 && uy < g.ny && iz >= 0 && iz < g.nz && q0 >= 0 && q1 + 1 <= g.nx &&
                                      (long long)ub0 + (long long)(q1 + 1) * g.nz < g.ntabB,
                                  "unit table index");
                        // 128-bit entries {start, prefixes}: the x-run ends' starts come with the prefixes
                        const int4 e0 = __ldg(tp + q0 * g.nz), e3 = __ldg(tp + (q1 + 1) * g.nz);
                        const int a0 = e0.x, a3 = e3.x;
                        if (kStats) ntab += 2u + (unsigned)(in && j0 != q0) + (unsigned)(in && j1 != q1);
                        int a1 = a3, a2 = a3;   // no inside run: [q0, q1] is tested whole
                        if (in) {
                            const int4 lo = j0 == q0 ? e0 : __ldg(tp + j0 * g.nz);
                            const int4 hi = j1 == q1 ? e3 : __ldg(tp + (j1 + 1) * g.nz);
                            // the modular differences are exact for runs of < 2^24 records: always when
                            // the map has fewer gain-eligible Gaussians (kLongRuns = false); otherwise a
                            // longer inside run is tested record by record instead
                            if (!kLongRuns || hi.x - lo.x < (1 << 24)) {
                            a1 = lo.x;
                            a2 = hi.x;
                            // differences of the packed prefixes, modulo 2^48 / 2^24 (exact: one x-run)
                            const unsigned long long qh = ((unsigned long long)((unsigned)hi.z & 0xffffu) << 32) | (unsigned)hi.y;
                            const unsigned long long ql = ((unsigned long long)((unsigned)lo.z & 0xffffu) << 32) | (unsigned)lo.y;
                            acc += (qh - ql) & 0xffffffffffffull;
                            const unsigned nhh = ((unsigned)hi.z >> 16) | (((unsigned)hi.w & 0xffu) << 16);
                            const unsigned nhl = ((unsigned)lo.z >> 16) | (((unsigned)lo.w & 0xffu) << 16);
                            acch += (int)((nhh - nhl) & 0xffffffu);
                            accl += (int)((((unsigned)hi.w >> 8) - ((unsigned)lo.w >> 8)) & 0xffffffu);
                            if (kStats) nagg += 1;
                            }
                        }
                        s0 = g.offB + a0;
                        l0 = a1 - a0;
                        s1 = g.offB + a2;
                        l1 = a3 - a2;
                    }
                    if (kStats) nunit += pos < U;
                    ub += 32;
                } else if (rnext <= iy1) {
                    // ---- row chunk: rows rnext .. rnext + 31, horizontal intervals
                    rcur = rnext;
                    rnext += 32;
                    const int iy = rcur + lane;
                    const float fiy = (float)iy;
                    if (kStats) nrow += iy <= iy1;
                    float plo = 0.f, phi = (float)(g.nx - 1), ilo = 0.f, ihi = phi;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const float4 C = sw.con[j];
                        cut(C, fmaf(C.y, fiy, C.x), plo, phi, ilo, ihi);
                    }
                    const int p0 = (int)fminf(plo, (float)g.nx);
                    const int p1 = iy <= iy1 ? (int)phi : -1;
                    ri0 = max((int)fminf(ilo, (float)g.nx), p0);
                    ri1 = min((int)ihi, p1);
                    int nu = 0, izlo = 0;
                    if (p0 <= p1) {
                        // flanks P \ I of copy A (one run when I is empty)
                        const int* sa = gstartA + iy * g.nx;
                        const bool in = ri0 <= ri1;
                        RTG_CHECK(iy >= 0 && iy < g.ny && p0 >= 0 && p1 + 1 <= g.nx &&
                                      (long long)iy * g.nx + p1 + 1 < g.ntabA,
                                  "flank table index");
                        s0 = __ldg(sa + p0);
                        l0 = __ldg(sa + (in ? ri0 : p1 + 1)) - s0;
                        if (kStats) nrowb += in ? 16u : 8u;   // copy-A column starts (4 bytes each)
                        if (in) {
                            s1 = __ldg(sa + ri1 + 1);
                            l1 = __ldg(sa + p1 + 1) - s1;
                            // z-cells the inside columns can see: vertical wedge at their largest
                            // depth, cut to the occupied z-range of the x-blocks they span
                            const float4 Cn = sw.con[0];
                            const float F0 = fmaf(Cn.y, fiy, Cn.x);
                            const float An = 1.0f / Cn.z;
                            const float Zmax =
                                fminf(fmaxf(fmaf(An, (float)ri0, F0), fmaf(An, (float)ri1, F0)) + Cn.w + g.zn,
                                      g.zf + g.eps);
                            const int zlo = fcell((zrel - g.kyd * Zmax - g.eps) * g.inv_hz, g.nz);
                            const int zhi = fcell((zrel + g.kyu * Zmax + g.eps) * g.inv_hz, g.nz);
                            int olo = INT_MAX, ohi = -1;
                            const int2* zo = zocc + iy * g.nxb;
                            RTG_CHECK(ri1 / kZoccX < g.nxb, "z-occupancy block");
                            // four blocks per step: the loads are issued before any is used
                            const int bend = ri1 / kZoccX;
                            for (int b = ri0 / kZoccX; b <= bend; b += 4) {
                                int2 o[4];
#pragma unroll
                                for (int u = 0; u < 4; ++u)
                                    o[u] = b + u <= bend ? __ldg(zo + b + u) : make_int2(INT_MAX, -1);
#pragma unroll
                                for (int u = 0; u < 4; ++u) {
                                    olo = min(olo, o[u].x);
                                    ohi = max(ohi, o[u].y);
                                }
                            }
                            if (kStats) nrowb += 8u * (unsigned)(bend - ri0 / kZoccX + 1);   // z-occupancy blocks
                            izlo = max(zlo, olo);
                            nu = max(0, min(zhi, ohi) - izlo + 1);
                        }
                        if (kStats) nflank += (unsigned long long)(l0 + l1);
                    }
                    incl = nu;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int v = __shfl_up_sync(kFullG, incl, o);
                        if (lane >= o) incl += v;
                    }
                    U = __shfl_sync(kFullG, incl, 31);
                    zoff = izlo - (incl - nu);
                    ub = 0;
                    if (U <= kMaxUnits) {
                        for (int u = incl - nu; u < incl; ++u) sw.owner[u] = (unsigned char)lane;
                        __syncwarp();
                    }
                } else {
                    done = true;
                }
                // ---- queue this lane's (<= 2) runs
                {
                    const bool c0 = l0 > 0, c1 = l1 > 0;
                    const unsigned b0 = __ballot_sync(kFullG, c0), b1 = __ballot_sync(kFullG, c1);
                    int slot = nq + __popc(b0 & lanes_lt) + __popc(b1 & lanes_lt);
                    if (c0) {
                        qs[slot] = s0;
                        qe[slot] = l0;
                        ++slot;
                    }
                    if (c1) {
                        qs[slot] = s1;
                        qe[slot] = l1;
                    }
                    nq += __popc(b0) + __popc(b1);
                    if (kStats) nruns += (unsigned)(__popc(b0) + __popc(b1));
                }
                if (nq > kQFlush || (done && nq > 0)) {
                    // ---- test every queued item, 64 per pass (two per lane)
                    __syncwarp();
                    int tot;
                    {
                        // items before each run (lane j: runs 8j .. 8j+7, then a warp scan); the
                        // start becomes start - items before, so item p of run r is record p + qs[r]
                        int4 la = *reinterpret_cast<const int4*>(qe + 8 * lane);
                        int4 lb = *reinterpret_cast<const int4*>(qe + 8 * lane + 4);
                        int4 sa = *reinterpret_cast<const int4*>(qs + 8 * lane);
                        int4 sb = *reinterpret_cast<const int4*>(qs + 8 * lane + 4);
                        const int r8 = nq - 8 * lane;   // runs of this lane that exist: min(8, max(0, r8))
                        if (r8 < 1) la.x = 0;
                        if (r8 < 2) la.y = 0;
                        if (r8 < 3) la.z = 0;
                        if (r8 < 4) la.w = 0;
                        if (r8 < 5) lb.x = 0;
                        if (r8 < 6) lb.y = 0;
                        if (r8 < 7) lb.z = 0;
                        if (r8 < 8) lb.w = 0;
                        const int sum = la.x + la.y + la.z + la.w + lb.x + lb.y + lb.z + lb.w;
                        int sc = sum;
#pragma unroll
                        for (int o = 1; o < 32; o <<= 1) {
                            const int v = __shfl_up_sync(kFullG, sc, o);
                            if (lane >= o) sc += v;
                        }
                        tot = __shfl_sync(kFullG, sc, 31);
                        int4 ea, eb;
                        ea.x = sc - sum;
                        ea.y = ea.x + la.x;
                        ea.z = ea.y + la.y;
                        ea.w = ea.z + la.z;
                        eb.x = ea.w + la.w;
                        eb.y = eb.x + lb.x;
                        eb.z = eb.y + lb.y;
                        eb.w = eb.z + lb.z;
                        sa.x -= ea.x; sa.y -= ea.y; sa.z -= ea.z; sa.w -= ea.w;
                        sb.x -= eb.x; sb.y -= eb.y; sb.z -= eb.z; sb.w -= eb.w;
                        *reinterpret_cast<int4*>(qs + 8 * lane) = sa;
                        *reinterpret_cast<int4*>(qs + 8 * lane + 4) = sb;
                        // a run of zero-length entries past the queue never starts inside a window
                        if (r8 < 1) ea.x = INT_MAX;
                        if (r8 < 2) ea.y = INT_MAX;
                        if (r8 < 3) ea.z = INT_MAX;
                        if (r8 < 4) ea.w = INT_MAX;
                        if (r8 < 5) eb.x = INT_MAX;
                        if (r8 < 6) eb.y = INT_MAX;
                        if (r8 < 7) eb.z = INT_MAX;
                        if (r8 < 8) eb.w = INT_MAX;
                        *reinterpret_cast<int4*>(qe + 8 * lane) = ea;   // items before each run
                        *reinterpret_cast<int4*>(qe + 8 * lane + 4) = eb;
                        // sentinel run nq from item tot on: NaN padding records (never visible, never
                        // ambiguous), so the passes need no per-item bound check
                        if (lane == 0) qs[nq] = g.nan_rec - tot;
                    }
                    int r0 = 0;   // run holding item gb
                    for (int gb0 = 0; gb0 < tot; gb0 += 64 * kFlushPasses) {   // 32-bit sums: flushed
                        const int gend = min(tot, gb0 + 64 * kFlushPasses);
                        // head bitmap of this chunk: bit b <=> a run (or the sentinel) starts at item gb0 + b + 1
                        __syncwarp();
                        {
                            const int4 ea = *reinterpret_cast<const int4*>(qe + 8 * lane);
                            const int4 eb = *reinterpret_cast<const int4*>(qe + 8 * lane + 4);
                            const unsigned span = (unsigned)(kHeadWords * 32);
                            auto mark = [&](int e) {   // bit e - 1 - gb0: the window needs no shift
                                const unsigned b = (unsigned)(e - 1 - gb0);
                                if (b < span) atomicOr(&sw.head[b >> 5], 1u << (b & 31));
                            };
                            mark(ea.x); mark(ea.y); mark(ea.z); mark(ea.w);
                            mark(eb.x); mark(eb.y); mark(eb.z); mark(eb.w);
                            if (lane == 0) mark(tot);
                        }
                        __syncwarp();
                        unsigned w = 0, pc = 0;
                        for (int gb = gb0; gb < gend; gb += 64) {
                            // head bit k of (hhi:hlo) <=> a run starts at item gb + k + 1 (bits gb - gb0 ..)
                            const int hw = (gb - gb0) >> 5;
                            RTG_CHECK(hw + 1 < kHeadWords, "head bitmap window");
                            const uint2 h01 = *reinterpret_cast<const uint2*>(sw.head + hw);
                            const unsigned hlo = h01.x, hhi = h01.y;
                            const int na = __popc(hlo);
                            const int gpa = gb + lane, gpb = gpa + 32;
                            const int gia = gpa + qs[r0 + __popc(hlo & lanes_lt)];
                            const int gib = gpb + qs[r0 + na + __popc(hhi & lanes_lt)];
                            RTG_CHECK(r0 + na + __popc(hhi) <= nq && nq < kQCap + 64, "queue run index");
                            RTG_CHECK(gia >= 0 && gia < g.nrec && gib >= 0 && gib < g.nrec, "record index");
                            const GRec Ga = grec[(unsigned)gia], Gb = grec[(unsigned)gib];
                            float guard_a, guard_b;
                            const float ma = vis_margin_xy(f, cam, Ga.x, Ga.y, Ga.z, guard_a);
                            const float mb = vis_margin_xy(f, cam, Gb.x, Gb.y, Gb.z, guard_b);
                            bool visa = ma >= 0.0f, visb = mb >= 0.0f;
                            const bool amba = fabsf(ma) < guard_a;
                            const bool ambb = fabsf(mb) < guard_b;
                            if (__any_sync(kFullG, amba || ambb)) {
                                if (amba) {
                                    visa = vis_decide64_cs(f.px, f.py, f.pz, sw.cs[0], sw.cs[1], Ga.x, Ga.y,
                                                           Ga.z, cam.cam64);
                                    ++nref;
                                }
                                if (ambb) {
                                    visb = vis_decide64_cs(f.px, f.py, f.pz, sw.cs[0], sw.cs[1], Gb.x, Gb.y,
                                                           Gb.z, cam.cam64);
                                    ++nref;
                                }
                            }
                            add_if(visa, w, Ga.uc, pc);
                            add_if(visb, w, Gb.uc, pc);
                            if (kStats) nvis += (unsigned)visa + (unsigned)visb;
                            r0 += na + __popc(hhi);
                        }
                        acc += w - (pc << kUqBits);
                        acch += pc & (kClsL - 1);
                        accl += pc / kClsL;
                        __syncwarp();
                        for (int j = lane; j < kHeadWords; j += 32) sw.head[j] = 0u;
                    }
                    if (kStats) ntest += (unsigned long long)tot;
                    nq = 0;
                    __syncwarp();
                }
                if (done) break;
            }
        }
        // warp totals (exact: integers below 2^53)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            acc += __shfl_xor_sync(kFullG, acc, o);
            acch += __shfl_xor_sync(kFullG, acch, o);
            accl += __shfl_xor_sync(kFullG, accl, o);
        }
        if (lane == 0) {
            wp_gq[i] = (long long)acc;
            wp_nh[i] = acch;
            wp_nl[i] = accl;
        }
    }
    if (kStats) {
        nref = __reduce_add_sync(kFullG, nref);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            ntest += __shfl_xor_sync(kFullG, ntest, o);
            nagg += __shfl_xor_sync(kFullG, nagg, o);
            nunit += __shfl_xor_sync(kFullG, nunit, o);
            nflank += __shfl_xor_sync(kFullG, nflank, o);
            nvis += __shfl_xor_sync(kFullG, nvis, o);
            nrow += __shfl_xor_sync(kFullG, nrow, o);
            nruns += __shfl_xor_sync(kFullG, nruns, o);
            ntab += __shfl_xor_sync(kFullG, ntab, o);
            nrowb += __shfl_xor_sync(kFullG, nrowb, o);
        }
        if (lane == 0) {
            if (nref) atomicAdd(&stats[1], (unsigned long long)nref);
            atomicAdd(&stats[2], ntest / 32);   // every lane counted the warp's items
            atomicAdd(&stats[3], nagg);
            atomicAdd(&stats[5], nflank);
            atomicAdd(&stats[6], nunit);
            atomicAdd(&stats[7], nvis);
            atomicAdd(&stats[8], nrow);
            atomicAdd(&stats[9], nruns / 32);   // warp-uniform: every lane counted the warp's runs
            atomicAdd(&stats[10], ntab);
            atomicAdd(&stats[11], nrowb);
        }
    }
}

// FP64 cos / sin of each listed waypoint's yaw, once (the gain kernel's warps would otherwise all
// evaluate the same FP64 sincos on every lane)
__global__ void k_wp_trig(const int* __restrict__ list, const int* __restrict__ count, const float* __restrict__ Yaw,
                          double2* __restrict__ trig) {
    const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (e >= *count) return;
    double sn, cs;
    sincos((double)Yaw[list[e]], &sn, &cs);
    trig[e] = make_double2(cs, sn);
}

int g_sms_g = 0, g_occ_g = 0;

}  // namespace

cudaError_t launch_gain_culled(rtg_map_s* m, rtg_traj_s* tr, const CamK& cam, const int* list, const int* count,
                               long long list_max, long long* wp_gq, int* wp_nh, int* wp_nl, int* counter,
                               unsigned long long* stats, cudaStream_t st) {
    if (m->n_gain == 0) {   // nothing is visible: zero sums
        cudaError_t e = cudaMemsetAsync(wp_gq, 0, sizeof(long long) * (size_t)tr->K * tr->T, st);
        if (e == cudaSuccess) e = cudaMemsetAsync(wp_nh, 0, sizeof(int) * (size_t)tr->K * tr->T, st);
        if (e == cudaSuccess) e = cudaMemsetAsync(wp_nl, 0, sizeof(int) * (size_t)tr->K * tr->T, st);
        return e;
    }
    if (!g_sms_g) {
        cudaDeviceGetAttribute(&g_sms_g, cudaDevAttrMultiProcessorCount, m->device);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_occ_g, k_gain_culled<false, false>, kWarpsG * 32, 0);
        if (g_occ_g < 1) g_occ_g = 1;
    }
    const GainGrid& gg = m->gg;
    GainK g;
    g.ox = gg.ox; g.oy = gg.oy; g.oz = gg.oz; g.hx = gg.hx; g.hy = gg.hy; g.hz = gg.hz;
    g.inv_hz = 1.0f / gg.hz;
    g.nx = gg.nx; g.ny = gg.ny; g.nz = gg.nz; g.nxb = gg.nxb;
    g.offB = (int)m->n_gain_pad;
    g.nrec = 2 * m->n_gain_pad;
    g.nan_rec = (int)m->n_gain;     // n_gain_pad >= n_gain + 64 (rtg_map.cu): copy A's NaN tail
    g.ntabB = (long long)gg.ny * (gg.nx + 1) * gg.nz;
    g.ntabA = gg.ncellsA + 1;
    // eps >> the FP32 error of a cell's centre value (a few ulps of the largest term: offsets of
    // at most the grid extent plus the distance of any waypoint to the grid origin)
    double ext = fabs(gg.ox) + fabs(gg.oy) + fabs(gg.oz) + gg.nx * (double)gg.hx + gg.ny * (double)gg.hy +
                 gg.nz * (double)gg.hz + cam.zmid + cam.zhalf;
    g.eps = (float)(1e-3 + 64.0 * ldexp(1.0, -24) * 2.0 * ext);
    g.zn = cam.zmid - cam.zhalf; g.zf = cam.zmid + cam.zhalf;
    g.kxl = cam.kxh - cam.kxc; g.kxr = cam.kxh + cam.kxc;
    g.kyu = cam.kyh + cam.kyc; g.kyd = cam.kyh - cam.kyc;
    g.kxh = cam.kxh;
    double2* trig = nullptr;
    cudaError_t et = dev_alloc((void**)&trig, sizeof(double2) * (size_t)(list_max > 0 ? list_max : 1), st);
    if (et != cudaSuccess) return et;
    if (list_max > 0)
        note_launch(), k_wp_trig<<<(unsigned)((list_max + 255) / 256), 256, 0, st>>>(list, count, tr->yaw, trig);
    long long blocks = (list_max + kWarpsG - 1) / kWarpsG;
    long long cap = (long long)g_sms_g * g_occ_g;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    // packed table prefixes are exact for x-runs of < 2^24 records, guaranteed below 2^24 records in all
    // (RTG_LONG_RUNS=1 forces the guarded variant: the parity tests run it on small maps)
    static const bool force_long = getenv("RTG_LONG_RUNS") && getenv("RTG_LONG_RUNS")[0] == '1';
    const bool long_runs = force_long || m->n_gain >= (1LL << 24);
#define RTG_GAIN_LAUNCH(S, LR)                                                                                  \
    note_launch(), k_gain_culled<S, LR><<<(unsigned)blocks, kWarpsG * 32, 0, st>>>(                             \
                       tr->x, tr->y, tr->z, tr->yaw, list, count, trig, m->grec, m->gstartA, m->zocc,          \
                       m->gtabP, g, cam, wp_gq, wp_nh, wp_nl, counter, stats)
    if (stats) {
        if (long_runs) RTG_GAIN_LAUNCH(true, true);
        else RTG_GAIN_LAUNCH(true, false);
    } else {
        if (long_runs) RTG_GAIN_LAUNCH(false, true);
        else RTG_GAIN_LAUNCH(false, false);
    }
#undef RTG_GAIN_LAUNCH
    cudaError_t e2 = cudaGetLastError();
    dev_free(trig, st);
    return e2;
}

}  // namespace rtg
