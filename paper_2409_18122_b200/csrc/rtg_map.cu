// rtg_map.cu -- map intake, packing, classification and grid construction.
//
//  a1  per Gaussian, in FP64: unit quaternion -> R, inflated semi-axes a_i = lambda_g s_i + r_robot
//      (P:298-302), M = diag(1/a) R^T (rows: principal axes scaled by 1/a_i), bounding radius
//      r_b = max_i a_i; stored as FP32 records (+ an FP64 copy of M for the re-decision branch).
//      Records are placed by a counting sort into two uniform grids:
//        * visibility grid: rows (hy) x x-cells (hx) x z-cells (hz), gain-eligible Gaussians only,
//          two copies: B sorted by (row, z-cell, x-cell) (x-contiguous z-slabs) with exact per-record
//          prefixes of u_q and the class counts, counting-sorted from the inputs; A sorted by (row,
//          x-cell, z-cell) (whole columns) derived from B by moving cell blocks in z-fastest order;
//        * collision grid: cubic cells (h), x fastest, collidable (non-ground) Gaussians only.
//  a2  classification over the gain-eligible set in ORIGINAL input order (deterministic FP64
//      two-pass mean / population std), class increments and exact fixed-point u per
//      record, and the exclusive prefixes over the records that let the culled kernel add whole x-runs.
#include <algorithm>
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "rtg_host.hpp"

namespace rtg {
namespace {

constexpr int kRedBlocks = 512;
constexpr int kRedThreads = 256;

__host__ __device__ inline int f2o(float f) {
#ifdef __CUDA_ARCH__
    int i = __float_as_int(f);
#else
    int i;
    std::memcpy(&i, &f, 4);
#endif
    return i >= 0 ? i : i ^ 0x7fffffff;
}
inline float o2f(int i) {
    int b = i >= 0 ? i : i ^ 0x7fffffff;
    float f;
    std::memcpy(&f, &b, 4);
    return f;
}

struct DevBounds {
    int err;
    int n_gain, n_col;
    int gmin[3], gmax[3], cmin[3], cmax[3];
    int rbmax, rhomax;
};

__global__ void k_bounds_init(DevBounds* b) {
    b->err = 0;
    b->n_gain = 0;
    b->n_col = 0;
    for (int i = 0; i < 3; ++i) {
        b->gmin[i] = b->cmin[i] = f2o(FLT_MAX);
        b->gmax[i] = b->cmax[i] = f2o(-FLT_MAX);
    }
    b->rbmax = f2o(0.f);
    b->rhomax = f2o(1.f);
}


struct BoundsAcc {
    int err = 0, ng = 0, nc = 0;
    int gmn[3] = {INT_MAX, INT_MAX, INT_MAX}, gmx[3] = {INT_MIN, INT_MIN, INT_MIN};
    int cmn[3] = {INT_MAX, INT_MAX, INT_MAX}, cmx[3] = {INT_MIN, INT_MIN, INT_MIN};
    int rbm = INT_MIN, rhm = INT_MIN;
};

// validation + bounds of one Gaussian's fp32 inputs
__device__ __forceinline__ void bounds_one(BoundsAcc& A, float px, float py, float pz, float q0, float q1, float q2,
                                           float q3, float s0, float s1, float s2, float op, float wi, unsigned f,
                                           const rtg_robot& rb) {
    const float p[3] = {px, py, pz};
    if (!(isfinite(px) && isfinite(py) && isfinite(pz))) A.err |= 1;
    double qn = (double)q0 * q0 + (double)q1 * q1 + (double)q2 * q2 + (double)q3 * q3;
    if (!(qn >= 1e-24) || !isfinite(qn)) A.err |= 2;
    if (!(s0 > 0.f && s1 > 0.f && s2 > 0.f) || !isfinite(s0) || !isfinite(s1) || !isfinite(s2)) A.err |= 4;
    if (!(wi >= 0.f) || !isfinite(wi)) A.err |= 8;
    if (!(op >= 0.f && op <= 1.f)) A.err |= 16;
    if (!(f & RTG_G_NO_GAIN)) {
        ++A.ng;
        for (int d = 0; d < 3; ++d) {
            int o = f2o(p[d]);
            A.gmn[d] = min(A.gmn[d], o);
            A.gmx[d] = max(A.gmx[d], o);
        }
    }
    if (!(f & RTG_G_NO_COLLIDE)) {
        ++A.nc;
        for (int d = 0; d < 3; ++d) {
            int o = f2o(p[d]);
            A.cmn[d] = min(A.cmn[d], o);
            A.cmx[d] = max(A.cmx[d], o);
        }
        double a[3];
        semi_axes64(s0, s1, s2, rb, a);
        double amax = fmax(a[0], fmax(a[1], a[2])), amin = fmin(a[0], fmin(a[1], a[2]));
        if (isfinite(amax)) {
            A.rbm = max(A.rbm, f2o(__double2float_ru(amax)));
            A.rhm = max(A.rhm, f2o(__double2float_ru(amax / amin)));
        }
    }
}

// one streaming pass over the inputs: validation, bounds, and the map's own copies of the weights
// and flags (w_out, flags_out); kVec: four consecutive Gaussians per step with 128-bit loads of every
// planar array (needs n % 4 == 0 and 16-byte aligned arrays)
template <bool kVec>
__global__ void k_bounds(long long n, const float* __restrict__ means, const float* __restrict__ quats,
                         const float* __restrict__ scales, const float* __restrict__ opacity,
                         const float* __restrict__ w, const unsigned char* __restrict__ flags, rtg_robot rb,
                         float* __restrict__ w_out, unsigned char* __restrict__ flags_out,
                         DevBounds* __restrict__ out) {
    BoundsAcc A;
    if (kVec) {
        const long long n4 = n >> 2;
        for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n4;
             j += (long long)gridDim.x * blockDim.x) {
            const float4 mx = __ldg(reinterpret_cast<const float4*>(means) + j);
            const float4 my = __ldg(reinterpret_cast<const float4*>(means + n) + j);
            const float4 mz = __ldg(reinterpret_cast<const float4*>(means + 2 * n) + j);
            const float4 qa = __ldg(reinterpret_cast<const float4*>(quats) + j);
            const float4 qb = __ldg(reinterpret_cast<const float4*>(quats + n) + j);
            const float4 qc = __ldg(reinterpret_cast<const float4*>(quats + 2 * n) + j);
            const float4 qd = __ldg(reinterpret_cast<const float4*>(quats + 3 * n) + j);
            const float4 sa = __ldg(reinterpret_cast<const float4*>(scales) + j);
            const float4 sb = __ldg(reinterpret_cast<const float4*>(scales + n) + j);
            const float4 sc = __ldg(reinterpret_cast<const float4*>(scales + 2 * n) + j);
            const float4 wv = __ldg(reinterpret_cast<const float4*>(w) + j);
            const float4 ov = opacity ? __ldg(reinterpret_cast<const float4*>(opacity) + j) : make_float4(.5f, .5f, .5f, .5f);
            const unsigned fv = flags ? __ldg(reinterpret_cast<const unsigned*>(flags) + j) : 0u;
            reinterpret_cast<float4*>(w_out)[j] = wv;
            if (flags) reinterpret_cast<unsigned*>(flags_out)[j] = fv;
            bounds_one(A, mx.x, my.x, mz.x, qa.x, qb.x, qc.x, qd.x, sa.x, sb.x, sc.x, ov.x, wv.x, fv & 0xffu, rb);
            bounds_one(A, mx.y, my.y, mz.y, qa.y, qb.y, qc.y, qd.y, sa.y, sb.y, sc.y, ov.y, wv.y, (fv >> 8) & 0xffu, rb);
            bounds_one(A, mx.z, my.z, mz.z, qa.z, qb.z, qc.z, qd.z, sa.z, sb.z, sc.z, ov.z, wv.z, (fv >> 16) & 0xffu, rb);
            bounds_one(A, mx.w, my.w, mz.w, qa.w, qb.w, qc.w, qd.w, sa.w, sb.w, sc.w, ov.w, wv.w, fv >> 24, rb);
        }
    } else {
        for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
             i += (long long)gridDim.x * blockDim.x) {
            const float wi = w[i];
            const unsigned f = flags ? flags[i] : 0u;
            w_out[i] = wi;
            if (flags) flags_out[i] = (unsigned char)f;
            bounds_one(A, means[i], means[n + i], means[2 * n + i], quats[i], quats[n + i], quats[2 * n + i],
                       quats[3 * n + i], scales[i], scales[n + i], scales[2 * n + i], opacity ? opacity[i] : 0.5f,
                       wi, f, rb);
        }
    }
    int err = A.err, ng = A.ng, nc = A.nc, rbm = A.rbm, rhm = A.rhm;
    int gmn[3], gmx[3], cmn[3], cmx[3];
    for (int d = 0; d < 3; ++d) {
        gmn[d] = A.gmn[d]; gmx[d] = A.gmx[d]; cmn[d] = A.cmn[d]; cmx[d] = A.cmx[d];
    }
    // warp aggregate, one atomic per warp
    unsigned full = 0xffffffffu;
    err = __reduce_or_sync(full, err);
    ng = __reduce_add_sync(full, ng);
    nc = __reduce_add_sync(full, nc);
    for (int d = 0; d < 3; ++d) {
        gmn[d] = __reduce_min_sync(full, gmn[d]);
        gmx[d] = __reduce_max_sync(full, gmx[d]);
        cmn[d] = __reduce_min_sync(full, cmn[d]);
        cmx[d] = __reduce_max_sync(full, cmx[d]);
    }
    rbm = __reduce_max_sync(full, rbm);
    rhm = __reduce_max_sync(full, rhm);
    // block aggregate through shared memory: one set of atomics per block
    __shared__ int sh[8][17];
    const int wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        int* s = sh[wid];
        s[0] = err; s[1] = ng; s[2] = nc;
        for (int d = 0; d < 3; ++d) {
            s[3 + d] = gmn[d]; s[6 + d] = gmx[d]; s[9 + d] = cmn[d]; s[12 + d] = cmx[d];
        }
        s[15] = rbm; s[16] = rhm;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    for (int w = 1; w < nw; ++w) {
        const int* s = sh[w];
        err |= s[0]; ng += s[1]; nc += s[2];
        for (int d = 0; d < 3; ++d) {
            gmn[d] = min(gmn[d], s[3 + d]); gmx[d] = max(gmx[d], s[6 + d]);
            cmn[d] = min(cmn[d], s[9 + d]); cmx[d] = max(cmx[d], s[12 + d]);
        }
        rbm = max(rbm, s[15]); rhm = max(rhm, s[16]);
    }
    {
        if (err) atomicOr(&out->err, err);
        if (ng) atomicAdd(&out->n_gain, ng);
        if (nc) atomicAdd(&out->n_col, nc);
        for (int d = 0; d < 3; ++d) {
            atomicMin(&out->gmin[d], gmn[d]);
            atomicMax(&out->gmax[d], gmx[d]);
            atomicMin(&out->cmin[d], cmn[d]);
            atomicMax(&out->cmax[d], cmx[d]);
        }
        atomicMax(&out->rbmax, rbm);
        atomicMax(&out->rhomax, rhm);
    }
}

// cell of coordinate v on a grid with origin o and inverse cell size ih (FP64; the culled kernels
// allow for eps around the cell boundaries, so ih may be rounded)
// layout maps: the rebuild's data must lie inside the caller's boxes and bounds (the grids were fixed by
// them), else the map is flagged (rtg_map_check): 32 gain-eligible mean outside, 64 collidable mean
// outside, 128 a_max above rb_max, 256 a_max / a_min above rho_max
__global__ void k_layout_check(DevBounds* __restrict__ b, rtg_map_layout L) {
    if (threadIdx.x != 0) return;
    int err = 0;
    if (b->n_gain > 0)
        for (int d = 0; d < 3; ++d)
            if (b->gmin[d] < f2o(L.gain_lo[d]) || b->gmax[d] > f2o(L.gain_hi[d])) err |= 32;
    if (b->n_col > 0) {
        for (int d = 0; d < 3; ++d)
            if (b->cmin[d] < f2o(L.col_lo[d]) || b->cmax[d] > f2o(L.col_hi[d])) err |= 64;
        if (b->rbmax > f2o(L.rb_max)) err |= 128;
        if (b->rhomax > f2o(L.rho_max)) err |= 256;
    }
    b->err |= err;
}

__device__ __forceinline__ int cell_coord(float v, double o, double ih, int nmax) {
    int c = (int)floor(((double)v - o) * ih);
    return c < 0 ? 0 : (c >= nmax ? nmax - 1 : c);
}

__global__ void k_zocc_init(int2* zocc, long long n) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < n) zocc[i] = make_int2(INT_MAX, -1);
}

// cell keys: visibility key (iy, iz, ix), collision key (iz, iy, ix); per-cell counts, each
// Gaussian's rank in its cells (the counting-sort slot within the cell, so the scatter needs no second
// atomic) and the occupied z-range of every row block
__global__ void k_keys(long long n, const float* __restrict__ means, const unsigned char* __restrict__ flags,
                       GainGrid gg, ColGrid cg, int* __restrict__ gkey, int* __restrict__ ckey,
                       int* __restrict__ grank, int* __restrict__ crank, int* __restrict__ gcountB,
                       int* __restrict__ gcountA, int2* __restrict__ zocc, int* __restrict__ ccount) {
    const double igx = 1.0 / gg.hx, igy = 1.0 / gg.hy, igz = 1.0 / gg.hz, icg = 1.0 / cg.h;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        float x = means[i], y = means[n + i], z = means[2 * n + i];
        unsigned f = flags ? flags[i] : 0u;
        int gk = -1, ck = -1;
        if (!(f & RTG_G_NO_GAIN)) {
            int ix = cell_coord(x, gg.ox, igx, gg.nx);
            int iy = cell_coord(y, gg.oy, igy, gg.ny);
            int iz = cell_coord(z, gg.oz, igz, gg.nz);
            gk = (int)(((long long)iy * gg.nz + iz) * gg.nx + ix);
            grank[i] = atomicAdd(&gcountB[gk], 1);
            if (gcountA) {   // scan path only (k_tabs_cols derives both from the cell starts)
                atomicAdd(&gcountA[(long long)iy * gg.nx + ix], 1);   // column totals (copy A), no rank needed
                int2* zo = zocc + (long long)iy * gg.nxb + ix / kZoccX;
                if (iz < zo->x) atomicMin(&zo->x, iz);
                if (iz > zo->y) atomicMax(&zo->y, iz);
            }
        }
        if (!(f & RTG_G_NO_COLLIDE)) {
            int ix = cell_coord(x, cg.ox, icg, cg.nx);
            int iy = cell_coord(y, cg.oy, icg, cg.ny);
            int iz = cell_coord(z, cg.oz, icg, cg.nz);
            ck = (int)(((long long)iz * cg.ny + iy) * cg.nx + ix);
            crank[i] = atomicAdd(&ccount[ck], 1);
        }
        gkey[i] = gk;
        ckey[i] = ck;
    }
}

__device__ __forceinline__ double u_of(float w, int variant) {
    double u = (double)w;
    return variant == RTG_VARIANT_SQ ? u * u : u;
}

// packed record word uc = u_q | c << 24 of a Gaussian with weight w (a2): class byte c =
// kClsH (u > tau_hi), kClsL (u < tau_lo), 0 (O); u_q = round(u 2^S) < 2^24
__device__ __forceinline__ unsigned class_of(float w, int variant, const ClassState* __restrict__ cs) {
    const double u = u_of(w, variant);
    const unsigned c = u > cs->tau_hi ? kClsH : (u < cs->tau_lo ? kClsL : 0u);
    return (unsigned)llrint(u * cs->scale) | (c << kUqBits);
}

// map build, per-cell tables by (row, kTabsX-column tile) (k_tabs_cols) up to kTabsMaxZ z-cells
constexpr int kTabsX = 2 * kZoccX;   // columns per CTA: two z-occupancy blocks
constexpr int kTabsMaxZ = 32;

// the record's (u_q, nH | nL << 32) pair added to the sum of its (z-slab, kTabsX-column tile) segment of copy B
// (fire-and-forget atomics; k_tabs_cols turns the scanned segment sums into the table's prefixes)
__device__ __forceinline__ void add_tile_sum(unsigned long long* __restrict__ tsum, int ntl, int nx, int key,
                                             unsigned uc) {
    const int slab = key / nx, tl = (key - slab * nx) / kTabsX;
    unsigned long long* t = tsum + 2 * ((long long)slab * ntl + tl);
    const unsigned q = uc & kUqMask, c = uc >> kUqBits;
    if (q) atomicAdd(t, (unsigned long long)q);
    if (c == kClsH) atomicAdd(t + 1, 1ull);
    else if (c == kClsL) atomicAdd(t + 1, 1ull << 32);
}

// large maps: the visibility records in two coalesced passes instead of the scatter above (whose
// partial 16-byte sectors cost read-modify-writes once the records exceed L2): (1) the permutation -- each
// eligible Gaussian writes its index into its slot; (2) every slot, in order, gathers its record, packed
// beforehand in input order with the class word (a2).  The scatter up to this many record bytes (r1,
// with two record copies: 64 MB scattered in 0.59 ms vs 0.67 ms gathered; 160 MB: 1.45 vs 1.23 ms)
constexpr double kScatterMaxBytes = 96.0 * 1024 * 1024;
constexpr double kScatterBothMaxBytes = 200.0 * 1024 * 1024;

__global__ void k_pack_gain(long long n, const float* __restrict__ means, const float* __restrict__ w,
                            GRec* __restrict__ rec, int variant, const ClassState* __restrict__ cs) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        rec[i] = GRec{means[i], means[n + i], means[2 * n + i], class_of(w[i], variant, cs)};
}

__global__ void k_perm_gain(long long n, const int* __restrict__ gkey, const int* __restrict__ grank,
                            const int* __restrict__ startB, int* __restrict__ gidx, const GRec* __restrict__ rec,
                            unsigned long long* __restrict__ tsum, int ntl, int nx) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const int k = gkey[i];
        if (k < 0) continue;
        gidx[startB[k] + grank[i]] = (int)i;
        if (tsum) add_tile_sum(tsum, ntl, nx, k, rec[i].uc);
    }
}

__global__ void k_fill_gain(long long n_gain, const int* __restrict__ dn_gain, const int* __restrict__ gidx,
                            const GRec* __restrict__ rec, GRec* __restrict__ grec) {
    const long long ng = dn_gain ? *dn_gain : n_gain;   // (a layout map: the device count)
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < ng;
         j += (long long)gridDim.x * blockDim.x)
        grec[j] = rec[gidx[j]];
}

// FP64 packing of the collision record (a1)
__device__ __forceinline__ void scatter_col_one(long long i, long long n, const float* __restrict__ means,
                                                const float* __restrict__ quats, const float* __restrict__ scales,
                                                int k, const int* __restrict__ crank, const int* __restrict__ cstart,
                                                const rtg_robot& rb, double guard, CRec* __restrict__ crec,
                                                CMat* __restrict__ cmat, CSrc* __restrict__ csrc) {
    const int slot = cstart[k] + crank[i];
    CSrc src;
    src.q[0] = quats[i]; src.q[1] = quats[n + i]; src.q[2] = quats[2 * n + i]; src.q[3] = quats[3 * n + i];
    src.s[0] = scales[i]; src.s[1] = scales[n + i]; src.s[2] = scales[2 * n + i];
    src.pad = 0.f;
    double a[3], M[9];
    pack_m64(src.q[0], src.q[1], src.q[2], src.q[3], src.s[0], src.s[1], src.s[2], rb, M, a);
    double amax = fmax(a[0], fmax(a[1], a[2]));
    float rb2 = __double2float_ru(amax * amax * (1.0 + guard) * (1.0 + 1.0e-6));
    crec[slot] = CRec{means[i], means[n + i], means[2 * n + i], rb2};
    CMat cm;
    for (int j = 0; j < 9; ++j) cm.m[j] = (float)M[j];
    cm.m[9] = __int_as_float((int)i);
    cm.m[10] = 0.f;
    cm.m[11] = 0.f;
    cmat[slot] = cm;
    csrc[slot] = src;
}

__global__ void k_scatter_col(long long n, const float* __restrict__ means, const float* __restrict__ quats,
                              const float* __restrict__ scales, const int* __restrict__ ckey,
                              const int* __restrict__ crank, const int* __restrict__ cstart, rtg_robot rb,
                              double guard, CRec* __restrict__ crec,
                              CMat* __restrict__ cmat, CSrc* __restrict__ csrc) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const int k = ckey[i];
        if (k >= 0) scatter_col_one(i, n, means, quats, scales, k, crank, cstart, rb, guard, crec, cmat, csrc);
    }
}

// both record scatters in one pass: the visibility records, sorted by (row, z-cell, x-cell), with their
// packed class and fixed-point u (the classification statistics are computed before) and their segment
// sums (tsum, or NULL), and the collision records as k_scatter_col: one read of the means and keys, both
// streams of random writes in flight together (crank NULL: the visibility records only)
__global__ void k_scatter_both(long long n, const float* __restrict__ means, const float* __restrict__ w,
                               const float* __restrict__ quats, const float* __restrict__ scales,
                               const int* __restrict__ gkey, const int* __restrict__ grank,
                               const int* __restrict__ startB, GRec* __restrict__ grec, int* __restrict__ gidx,
                               int variant, const ClassState* __restrict__ cs, unsigned long long* __restrict__ tsum,
                               int ntl, int nx, const int* __restrict__ ckey, const int* __restrict__ crank,
                               const int* __restrict__ cstart, rtg_robot rb, double guard, CRec* __restrict__ crec,
                               CMat* __restrict__ cmat, CSrc* __restrict__ csrc) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const int k = gkey[i], kc = crank ? ckey[i] : -1;
        if (k >= 0) {
            const GRec r{means[i], means[n + i], means[2 * n + i], class_of(w[i], variant, cs)};
            const int sb = startB[k] + grank[i];
            grec[sb] = r;
            gidx[sb] = (int)i;
            if (tsum) add_tile_sum(tsum, ntl, nx, k, r.uc);
        }
        if (kc >= 0) scatter_col_one(i, n, means, quats, scales, kc, crank, cstart, rb, guard, crec, cmat, csrc);
    }
}

// copy A from copy B: copy A is sorted by (iy, x, iz), so column (iy, x) starts at gstartA (the
// exclusive scan of the column counts) and holds its cells (iy, iz, x) in iz order, each a contiguous
// block of copy B at tabB[(iy, x, iz)]; one thread per column moves them
// map build: the cells' copy-B starts and counts in key order [ny][nz][nx] (coalesced over x)
__global__ void k_derive_cols_b(long long ncols, int nx, int nz, const int* __restrict__ startB,
                                const int* __restrict__ countB, const int* __restrict__ gstartA,
                                const GRec* __restrict__ recB, GRec* __restrict__ recA) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;   // grid: x = columns of one row, y = rows
    if (x >= nx) return;
    const long long iy = blockIdx.y, col = iy * nx + x;
    const long long k0 = iy * nz * (long long)nx + x;
    int dst = gstartA[col];
    for (int iz = 0; iz < nz; ++iz) {
        const int src = startB[k0 + (long long)iz * nx], c = countB[k0 + (long long)iz * nx];
        for (int k = 0; k < c; ++k) recA[dst++] = recB[src + k];
    }
}

__global__ void k_derive_cols(long long ncols, int nx, int nz, const int* __restrict__ tabB,
                              const int* __restrict__ gstartA, const GRec* __restrict__ recB,
                              GRec* __restrict__ recA) {
    const long long col = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (col >= ncols) return;
    const long long iy = col / nx, x = col - iy * nx;
    const int* t = tabB + (iy * (nx + 1) + x) * nz * 4;   // 4-int TabP entries, start first
    int dst = gstartA[col];
    for (int iz = 0; iz < nz; ++iz) {
        const int src = t[iz * 4], end = t[(nz + iz) * 4];
        for (int k = src; k < end; ++k) recA[dst++] = recB[k];
    }
}

// NaN padding of the visibility records [g0, gto) of both copies (gidx -1) and of the collision records
// [c0, cto) in one launch, g0 / c0 the device counts when given (a layout map's rebuild: grid-stride from
// there, so a rebuild that fills its capacity pads nothing).  Only the collision record's sphere
// {NaN, -1} is written: the matrix and FP32 sources are read only after a passed sphere test.
__global__ void k_pad_records(GRec* __restrict__ recA, GRec* __restrict__ recB, int* __restrict__ gidx,
                              long long gfrom, long long gto, const int* __restrict__ dg, CRec* __restrict__ crec,
                              long long cfrom, long long cto, const int* __restrict__ dc) {
    const long long g0 = dg ? max(gfrom, (long long)*dg) : gfrom;
    const long long c0 = dc ? max(cfrom, (long long)*dc) : cfrom;
    const long long stride = (long long)gridDim.x * blockDim.x, t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const float nan = __int_as_float(0x7fc00000);
    for (long long i = g0 + t; i < gto; i += stride) {
        recB[i] = GRec{nan, nan, nan, 0u};
        recA[i] = GRec{nan, nan, nan, 0u};
        gidx[i] = -1;
    }
    for (long long i = c0 + t; i < cto; i += stride) crec[i] = CRec{nan, nan, nan, -1.f};
}

// ------------------------------------------------------------------ classification (a2)


// deterministic block tree over a fixed contiguous chunk
__device__ double block_sum(double v, double* sh) {
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
        __syncthreads();
    }
    double r = sh[0];
    __syncthreads();
    return r;
}

// pass 1: partial sums of u, counts and max u over eligible Gaussians, original order
__global__ void k_red1(long long n, const float* __restrict__ w, const unsigned char* __restrict__ flags,
                       int variant, double* __restrict__ part) {
    __shared__ double sh[kRedThreads];
    long long chunk = (n + gridDim.x - 1) / gridDim.x;
    long long lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
    double s = 0.0, c = 0.0, mx = 0.0;
    for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        if (flags && (flags[i] & RTG_G_NO_GAIN)) continue;
        double u = u_of(w[i], variant);
        s += u;
        c += 1.0;
        mx = fmax(mx, u);
    }
    double S = block_sum(s, sh);
    double C = block_sum(c, sh);
    sh[threadIdx.x] = mx;
    __syncthreads();
    for (int st = blockDim.x / 2; st > 0; st >>= 1) {
        if ((int)threadIdx.x < st) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + st]);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[3 * blockIdx.x + 0] = S;
        part[3 * blockIdx.x + 1] = C;
        part[3 * blockIdx.x + 2] = sh[0];
    }
}

__global__ void k_red1_final(const double* __restrict__ part, int nparts, ClassState* cs) {
    __shared__ double sh[kRedThreads];
    double s = 0.0, c = 0.0, mx = 0.0;
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) {
        s += part[3 * i];
        c += part[3 * i + 1];
        mx = fmax(mx, part[3 * i + 2]);
    }
    double S = block_sum(s, sh);
    double C = block_sum(c, sh);
    sh[threadIdx.x] = mx;
    __syncthreads();
    for (int st = blockDim.x / 2; st > 0; st >>= 1) {
        if ((int)threadIdx.x < st) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + st]);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        cs->n_eligible = (int)C;
        cs->mean = C > 0 ? S / C : 0.0;
        cs->std = sh[0];   // temporarily holds max u (consumed by k_red2_final)
    }
}

// pass 2: partial sums of (u - mean)^2
__global__ void k_red2(long long n, const float* __restrict__ w, const unsigned char* __restrict__ flags,
                       int variant, const ClassState* __restrict__ cs, double* __restrict__ part) {
    __shared__ double sh[kRedThreads];
    double m = cs->mean;
    long long chunk = (n + gridDim.x - 1) / gridDim.x;
    long long lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
    double s = 0.0;
    for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        if (flags && (flags[i] & RTG_G_NO_GAIN)) continue;
        double d = u_of(w[i], variant) - m;
        s += d * d;
    }
    double S = block_sum(s, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = S;
}

__global__ void k_red2_final(const double* __restrict__ part, int nparts, ClassState* cs, double k_sigma,
                             double tau_hi, double tau_lo, int has_hi, int has_lo) {
    __shared__ double sh[kRedThreads];
    double s = 0.0;
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += part[i];
    double S = block_sum(s, sh);
    if (threadIdx.x == 0) {
        double umax = cs->std;
        double cnt = (double)cs->n_eligible;
        double sd = cnt > 0 ? sqrt(S / cnt) : 0.0;
        cs->std = sd;
        cs->tau_hi = has_hi ? tau_hi : cs->mean + k_sigma * sd;
        cs->tau_lo = has_lo ? tau_lo : cs->mean - k_sigma * sd;
        int shift = 0;
        double tot = cnt * umax;
        if (tot > 0.0) {
            // sum of all u_q < 2^53 (exact in FP64) and every u_q < 2^24 (packed with the class)
            shift = (int)floor(fmin(52.0 - log2(tot), (double)(kUqBits - 1) - log2(umax)));
            shift = shift > 1000 ? 1000 : (shift < -1000 ? -1000 : shift);
        }
        cs->shift = shift;
        cs->scale = ldexp(1.0, shift);
        cs->inv_scale = ldexp(1.0, -shift);
    }
}

// class increments and fixed-point u per visibility record (both copies); copy B also
// writes u_q and the packed class count for its exact prefixes
__global__ void k_class_records(long long n_rec, GRec* __restrict__ grec, const int* __restrict__ gidx,
                                const float* __restrict__ w, int variant, const ClassState* __restrict__ cs) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n_rec) return;
    const int g = gidx[i];
    if (g < 0) return;
    grec[i].uc = class_of(w[g], variant, cs);
}


// one z-fastest table entry: the cell's first copy-B record and the exclusive prefixes there, modulo
// 2^48 (sum of u_q) and 2^24 (n_H, n_L) -- the culled kernel only takes differences of two entries of
// one (row, z-slab), exact while such an x-run holds fewer than 2^24 records (u_q < 2^24)
__device__ __forceinline__ TabP pack_tab(int start, const longlong2 v) {
    const unsigned long long q = (unsigned long long)v.x;
    const unsigned nh = (unsigned)(v.y & 0xffffff), nl = (unsigned)((v.y >> 32) & 0xffffff);
    TabP t;
    t.start = start;
    t.qlo = (unsigned)q;
    t.qhi_nh = (unsigned)((q >> 32) & 0xffff) | (nh << 16);
    t.nh_nl = (nh >> 16) | (nl << 8);
    return t;
}

// both z-fastest tables in one pass at map build: the copy-B start of the cell (key order scan)
// and the exact prefixes there
// (grid: x = entries of one row, y = rows, so the index arithmetic is 32-bit within a row)
__global__ void k_build_tabs(GainGrid gg, const int* __restrict__ startB, const longlong2* __restrict__ pqhl,
                             TabP* __restrict__ tabP) {
    const int er = blockIdx.x * blockDim.x + threadIdx.x;   // entry within the row: (ix, iz), iz fastest
    const int nrow = (gg.nx + 1) * gg.nz;
    if (er >= nrow) return;
    const long long iy = blockIdx.y;
    const int ix = er / gg.nz, iz = er - ix * gg.nz;
    const int s = startB[(iy * gg.nz + iz) * gg.nx + ix];
    tabP[iy * nrow + er] = pack_tab(s, pqhl[s]);
}

// the same through shared memory: a CTA takes tx columns of one row over all z-cells, reads the
// key-order starts and gathers the prefixes x-fastest (neighbouring cells share or neighbour their
// starts: coalesced), and stores the entries z-fastest (one contiguous range)
constexpr int kTabEntries = 1536;   // entries per CTA (24 KB of shared memory)
__global__ void __launch_bounds__(256) k_build_tabs_tile(GainGrid gg, int tx, const int* __restrict__ startB,
                                                         const longlong2* __restrict__ pqhl,
                                                         TabP* __restrict__ tabP) {
    __shared__ TabP sm[kTabEntries];
    const long long iy = blockIdx.y;
    const int x0 = blockIdx.x * tx, nz = gg.nz;
    const int ncol = min(tx, gg.nx + 1 - x0);
    for (int t = threadIdx.x; t < ncol * nz; t += blockDim.x) {
        const int iz = t / ncol, xl = t - iz * ncol;
        const int s = startB[(iy * nz + iz) * gg.nx + x0 + xl];   // x = nx: the slab's end
        sm[xl * nz + iz] = pack_tab(s, pqhl[s]);
    }
    __syncthreads();
    TabP* out = tabP + (iy * (gg.nx + 1) + x0) * nz;
    for (int t = threadIdx.x; t < ncol * nz; t += blockDim.x) out[t] = sm[t];
}

// map build, the per-cell tables in one pass per (row, kTabsX-column tile), from the cell starts (key
// order) and the scanned sums of the tile's z-slab segments of copy B:
//  - copy A's column starts: the row's first record plus, per z-slab, the slab's records left of the
//    column (rows and slabs are contiguous in copy B);
//  - copy A: each cell's records moved to their column, z-cells in order (what k_derive_cols_b does),
//    one record per thread over the tile's slab segments (coalesced reads; a cell's records are found
//    by binary search in the starts, so dense cells do not serialise a thread);
//  - the z-fastest entries {start, exact prefixes} (what the record prefix scan + k_build_tabs* do):
//    the segment's scanned base plus the sums of the cells to its left, stored as one contiguous range;
//  - the tile's z-occupancy block (what the key pass's atomics do on the other path).
// The map it builds is identical to the other path's.  nz <= kTabsMaxZ.
constexpr int kTabsThreads = 256;
static_assert(kTabsThreads > kTabsX && kTabsX % kZoccX == 0 && kTabsX % 32 == 0, "tile shape");
// shared-memory rows of kTabsX + 1 (odd) elements: a warp's accesses along z (the z-fastest entries)
// fall in distinct banks; the 16-byte sums are further skewed by one slot per 4 columns (kTabsSW, odd)
// so that lanes taking 4 consecutive columns each (the per-slab prefix) do too
constexpr int kTabsW = kTabsX + 1;
constexpr int kTabsSW = kTabsX + kTabsX / 4 + 1;
__device__ __forceinline__ int tabs_sx(int iz, int j) { return iz * kTabsSW + j + (j >> 2); }
inline size_t tabs_smem(int nz) {
    return sizeof(unsigned long long) * 2 * nz * kTabsSW  // per cell (u, nH | nL << 32), then its prefix
           + sizeof(longlong2) * nz                      // the slab segments' scanned bases
           + sizeof(int) * nz * kTabsW                   // cell starts
           + sizeof(int) * nz * kTabsX                   // cells' first copy-A slot
           + sizeof(int) * (2 * nz + 1);                 // slab starts, flattened segment offsets
}
__global__ void __launch_bounds__(kTabsThreads, 6) k_tabs_cols(GainGrid gg, int ntl, const int* __restrict__ startB,
                                                            const longlong2* __restrict__ tpre,
                                                            const GRec* __restrict__ recB, GRec* __restrict__ recA,
                                                            TabP* __restrict__ tabP, int* __restrict__ gstartA,
                                                            int2* __restrict__ zocc) {
    extern __shared__ __align__(16) unsigned char smraw[];
    __shared__ int s_zlo[kTabsX / kZoccX], s_zhi[kTabsX / kZoccX];
    const int nx = gg.nx, nz = gg.nz, tile = blockIdx.x, x0 = tile * kTabsX;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    constexpr int W = kTabsW;
    ulonglong2* s_sum = reinterpret_cast<ulonglong2*>(smraw);                     // [nz][kTabsSW], skewed
    longlong2* s_base = reinterpret_cast<longlong2*>(s_sum + nz * kTabsSW);        // [nz]
    int* s_st = reinterpret_cast<int*>(s_base + nz);                              // [nz][W]
    int* s_dA = s_st + nz * W;                                                    // [nz][kTabsX]
    int* s_slab0 = s_dA + nz * kTabsX;                                            // [nz]
    int* s_seg = s_slab0 + nz;                                                    // [nz + 1]
    const long long iy = blockIdx.y;
    const int ncol = max(0, min(kTabsX, nx - x0));   // columns of the tile
    const int nent = min(kTabsX, nx + 1 - x0);       // its table entries (x = nx: the slabs' ends)
    const long long kb = iy * nz * (long long)nx;    // key of cell (iy, 0, 0)
    if (threadIdx.x < kTabsX / kZoccX) {
        s_zlo[threadIdx.x] = INT_MAX;
        s_zhi[threadIdx.x] = -1;
    }
    // a warp per z-slab: its cell starts (coalesced, all loads in flight before the first use), the
    // slab start and scanned base
    constexpr int kLd = (kTabsX + 1 + 31) / 32;
    for (int iz = wid; iz < nz; iz += nw) {
        const int* src = startB + kb + (long long)iz * nx + x0;
        int v[kLd];
#pragma unroll
        for (int c = 0; c < kLd; ++c) v[c] = lane + 32 * c <= ncol ? __ldg(src + lane + 32 * c) : 0;
        int s0 = 0;
        longlong2 bs = make_longlong2(0, 0);
        if (lane == 0) {
            s0 = __ldg(startB + kb + (long long)iz * nx);
            bs = tpre[((long long)iy * nz + iz) * ntl + tile];
        }
#pragma unroll
        for (int c = 0; c < kLd; ++c)
            if (lane + 32 * c <= ncol) s_st[iz * W + lane + 32 * c] = v[c];
        if (lane == 0) {
            s_slab0[iz] = s0;
            s_base[iz] = bs;
        }
    }
    __syncthreads();
    if (threadIdx.x <= ncol) {
        const int j = threadIdx.x;
        int a = s_slab0[0];
        for (int iz = 0; iz < nz; ++iz) a += s_st[iz * W + j] - s_slab0[iz];
        gstartA[iy * nx + x0 + j] = a;   // j = ncol: the next column's start (its tile writes the same)
        if (j < ncol) {
            int zlo = INT_MAX, zhi = -1;
            for (int iz = 0; iz < nz; ++iz) {
                s_dA[iz * kTabsX + j] = a;
                s_sum[tabs_sx(iz, j)] = make_ulonglong2(0ull, 0ull);
                const int c = s_st[iz * W + j + 1] - s_st[iz * W + j];
                a += c;
                if (c > 0) {
                    zlo = min(zlo, iz);
                    zhi = iz;
                }
            }
            if (zhi >= 0) {
                atomicMin(&s_zlo[j / kZoccX], zlo);
                atomicMax(&s_zhi[j / kZoccX], zhi);
            }
        }
    } else if (threadIdx.x == blockDim.x - 1) {
        int o = 0;
        for (int iz = 0; iz < nz; ++iz) {
            s_seg[iz] = o;
            o += s_st[iz * W + ncol] - s_st[iz * W];
        }
        s_seg[nz] = o;
    }
    __syncthreads();
    // records, one per thread over the tile's slab segments: moved to copy A and summed per cell
    const int total = s_seg[nz];
    for (int fb = threadIdx.x - lane; fb < total; fb += blockDim.x) {   // warp-uniform trip count
        const int f = fb + lane;
        int cell = -1;
        unsigned q = 0u, hl = 0u;
        if (f < total) {
            int iz = 0;   // the slab: the last with s_seg[iz] <= f (empty slabs share their offset)
            for (int lo = 0, hi = nz - 1; lo < hi;) {
                const int mid = (lo + hi + 1) >> 1;
                if (s_seg[mid] <= f) lo = mid; else hi = mid - 1;
                iz = lo;
            }
            const int* st = s_st + iz * W;
            const int k = st[0] + (f - s_seg[iz]);
            int j = 0;    // the cell: the last with st[j] <= k
            for (int lo = 0, hi = ncol - 1; lo < hi;) {
                const int mid = (lo + hi + 1) >> 1;
                if (st[mid] <= k) lo = mid; else hi = mid - 1;
                j = lo;
            }
            const GRec r = recB[k];
            recA[s_dA[iz * kTabsX + j] + (k - st[j])] = r;
            const unsigned c = r.uc >> kUqBits;
            cell = tabs_sx(iz, j);
            q = r.uc & kUqMask;
            hl = c == kClsH ? 1u : (c == kClsL ? 0x10000u : 0u);
        }
        // a cell's records sit in consecutive lanes (cells ascend with f): segmented sums (exact, < 2^29
        // and < 2^16 per warp), one shared-memory add per cell and warp by the segment's last lane
        const int prev = __shfl_up_sync(0xffffffffu, cell, 1), next = __shfl_down_sync(0xffffffffu, cell, 1);
        const unsigned heads = __ballot_sync(0xffffffffu, lane == 0 || prev != cell);
        const int seg0 = 31 - __clz(heads & (0xffffffffu >> (31 - lane)));   // this lane's segment head
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned pq = __shfl_up_sync(0xffffffffu, q, o), ph = __shfl_up_sync(0xffffffffu, hl, o);
            if (lane - o >= seg0) {
                q += pq;
                hl += ph;
            }
        }
        if (cell >= 0 && (lane == 31 || next != cell)) {
            unsigned long long* sm = reinterpret_cast<unsigned long long*>(s_sum + cell);
            if (q) atomicAdd(sm, (unsigned long long)q);
            if (hl) atomicAdd(sm + 1, (unsigned long long)(hl & 0xffffu) | ((unsigned long long)(hl >> 16) << 32));
        }
    }
    __syncthreads();
    // exclusive prefixes along x within each z-slab from the segment's base (a warp per slab, 4
    // consecutive columns per lane summed serially, one warp scan of the lane totals)
    static_assert(kTabsX == 128, "4 columns per lane");
    for (int iz = wid; iz < nz; iz += nw) {
        ulonglong2 v[4];
        unsigned long long a = 0ull, b = 0ull;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int j = 4 * lane + i;
            v[i] = j < ncol ? s_sum[tabs_sx(iz, j)] : make_ulonglong2(0ull, 0ull);
            a += v[i].x;
            b += v[i].y;
        }
        const unsigned long long ta = a, tb = b;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long pa = __shfl_up_sync(0xffffffffu, a, o), pb = __shfl_up_sync(0xffffffffu, b, o);
            if (lane >= o) {
                a += pa;
                b += pb;
            }
        }
        unsigned long long ea = (unsigned long long)s_base[iz].x + a - ta,
                           eb = (unsigned long long)s_base[iz].y + b - tb;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int j = 4 * lane + i;
            if (j < nent) s_sum[tabs_sx(iz, j)] = make_ulonglong2(ea, eb);
            ea += v[i].x;
            eb += v[i].y;
        }
    }
    __syncthreads();
    // the z-fastest entries (iy, x0 .. x0 + nent - 1, all z): one contiguous range; t -> (j, iz) by a
    // float reciprocal (exact: t < 2^13, and t / nz is at least 1 / nz from the next integer)
    TabP* out = tabP + (iy * (nx + 1) + x0) * nz;
    const float rnz = 1.0f / (float)nz;
    for (int t = threadIdx.x; t < nent * nz; t += blockDim.x) {
        const int j = (int)(((float)t + 0.5f) * rnz), iz = t - j * nz;
        const ulonglong2 v = s_sum[tabs_sx(iz, j)];
        out[t] = pack_tab(s_st[iz * W + j], make_longlong2((long long)v.x, (long long)v.y));
    }
    if (threadIdx.x < kTabsX / kZoccX && x0 + threadIdx.x * kZoccX < nx)
        zocc[iy * gg.nxb + tile * (kTabsX / kZoccX) + threadIdx.x] = make_int2(s_zlo[threadIdx.x], s_zhi[threadIdx.x]);
}

// reclassification: new prefixes at every z-fastest table entry (its start unchanged)
__global__ void k_pack_tabP(long long nt, const longlong2* __restrict__ pqhl, TabP* __restrict__ tabP) {
    long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (e >= nt) return;
    const int t = tabP[e].start;   // the starts stay; the prefixes follow the new classes
    tabP[e] = pack_tab(t, pqhl[t]);
}

inline unsigned nblocks(long long n, int t) {
    long long b = (n + t - 1) / t;
    return (unsigned)(b < 1 ? 1 : (b > 65535LL * 32 ? 65535LL * 32 : b));
}

}  // namespace

// a2 statistics over the gain-eligible Gaussians in input order (deterministic FP64 two-pass
// mean / population std) -> thresholds and fixed-point scale in cls
static cudaError_t class_stats(long long n, const float* w, const unsigned char* flags, int variant, double k_sigma,
                               double tau_hi, double tau_lo, ClassState* cls, double* scratch, cudaStream_t st) {
    const bool has_hi = !std::isnan(tau_hi), has_lo = !std::isnan(tau_lo);
    const int nparts = kRedBlocks;
    note_launch(), k_red1<<<nparts, kRedThreads, 0, st>>>(n, w, flags, variant, scratch);
    note_launch(), k_red1_final<<<1, kRedThreads, 0, st>>>(scratch, nparts, cls);
    note_launch(), k_red2<<<nparts, kRedThreads, 0, st>>>(n, w, flags, variant, cls, scratch);
    note_launch(), k_red2_final<<<1, kRedThreads, 0, st>>>(scratch, nparts, cls, k_sigma, tau_hi, tau_lo, has_hi, has_lo);
    return cudaGetLastError();
}

// copy A (and gstartA) from copy B and its start table, in z-fastest cell order (map build and every
// reclassification: copy A carries the class words too)
static cudaError_t derive_copy_a(rtg_map_s* m, cudaStream_t st, const int* startB = nullptr,
                                 const int* countB = nullptr) {
    if (m->n_gain <= 0) return cudaSuccess;
    const GainGrid& gg = m->gg;
    const long long ncols = gg.ncellsA;
    const GRec* recB = m->grec + m->n_gain_pad;
    cudaError_t e = cudaSuccess;
    if (startB && countB) {   // map build: gstartA is scanned from the column counts; cell starts at hand
        note_launch(), k_derive_cols_b<<<dim3((unsigned)((gg.nx + 255) / 256), (unsigned)gg.ny), 256, 0, st>>>(
                           ncols, gg.nx, gg.nz, startB, countB, m->gstartA, recB, m->grec);
    } else {                  // reclassification: the starts from the table entries
        const int* tab = reinterpret_cast<const int*>(m->gtabP);   // TabP::start leads each 4-int entry
        e = exclusive_scan_col_counts(tab, 4, gg.nx, gg.nz, ncols, m->gstartA, st);
        if (e != cudaSuccess) return e;
        note_launch(), k_derive_cols<<<nblocks(ncols, 256), 256, 0, st>>>(ncols, gg.nx, gg.nz, tab, m->gstartA,
                                                                          recB, m->grec);
    }
    return cudaGetLastError();
}

// exact prefixes of copy B's (u_q, packed class count) pairs, gathered at the table entries
// startB (map build only): the key-order start table; the entries' starts are written in the same pass
static cudaError_t class_prefix(rtg_map_s* m, cudaStream_t st, const int* startB = nullptr,
                                const int* countB = nullptr) {
    const long long ng = m->n_gain;
    long long* pqhl = nullptr;
    cudaError_t e = dev_alloc((void**)&pqhl, 2 * sizeof(long long) * (ng + 1), st);
    if (e != cudaSuccess) return e;
    e = exclusive_scan_grec_uc(m->grec + m->n_gain_pad, pqhl, ng, st);
    if (e == cudaSuccess) {
        const long long nt = (long long)m->gg.ny * (m->gg.nx + 1) * m->gg.nz;
        if (startB)
        {
            const int tx = kTabEntries / m->gg.nz;
            if (tx >= 8)
                note_launch(), k_build_tabs_tile<<<dim3((unsigned)((m->gg.nx + 1 + tx - 1) / tx), (unsigned)m->gg.ny),
                                                   256, 0, st>>>(m->gg, tx, startB, (const longlong2*)pqhl, m->gtabP);
            else
                note_launch(), k_build_tabs<<<dim3((unsigned)(((m->gg.nx + 1) * m->gg.nz + 255) / 256),
                                                   (unsigned)m->gg.ny), 256, 0, st>>>(m->gg, startB,
                                                                                      (const longlong2*)pqhl, m->gtabP);
        }
        else
            note_launch(), k_pack_tabP<<<nblocks(nt, 256), 256, 0, st>>>(nt, (const longlong2*)pqhl, m->gtabP);
        e = cudaGetLastError();
    }
    dev_free(pqhl, st);
    if (e == cudaSuccess) e = derive_copy_a(m, st, startB, countB);
    return e;
}

static void set_class_params(rtg_map_s* m, int variant, double k_sigma, double tau_hi, double tau_lo) {
    m->cls_variant = variant;
    m->cls_k = k_sigma;
    m->cls_th_nan = std::isnan(tau_hi);
    m->cls_tl_nan = std::isnan(tau_lo);
    m->cls_th = tau_hi;
    m->cls_tl = tau_lo;
}

rtg_status classify_map(rtg_map_s* m, int variant, double k_sigma, double tau_hi, double tau_lo,
                        cudaStream_t st, bool force) {
    bool has_hi = !std::isnan(tau_hi), has_lo = !std::isnan(tau_lo);
    if (!force && m->cls_variant == variant && m->cls_k == k_sigma && m->cls_th_nan == !has_hi &&
        m->cls_tl_nan == !has_lo && (!has_hi || m->cls_th == tau_hi) && (!has_lo || m->cls_tl == tau_lo))
        return RTG_OK;
    cudaError_t e = class_stats(m->n, m->w_orig, m->flags, variant, k_sigma, tau_hi, tau_lo, m->cls, m->red_scratch, st);
    const long long nrec = m->n_gain_pad;   // copy B (copy A is re-derived by class_prefix)
    if (e == cudaSuccess && m->n_gain > 0) {
        note_launch(), k_class_records<<<nblocks(nrec, 256), 256, 0, st>>>(nrec, m->grec + m->n_gain_pad, m->gidx,
                                                                           m->w_orig, variant,
                                                                           m->cls);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = class_prefix(m, st);
    if (e != cudaSuccess) {
        set_error("classify: %s", cudaGetErrorString(e));
        return e == cudaErrorMemoryAllocation ? RTG_ERR_OUT_OF_MEMORY : RTG_ERR_CUDA;
    }
    set_class_params(m, variant, k_sigma, tau_hi, tau_lo);
    return RTG_OK;
}

#define MAP_CK(expr)                                                              \
    do {                                                                          \
        cudaError_t e_ = (expr);                                                  \
        if (e_ != cudaSuccess) {                                                  \
            set_error("%s: %s", #expr, cudaGetErrorString(e_));                   \
            return e_ == cudaErrorMemoryAllocation ? RTG_ERR_OUT_OF_MEMORY : RTG_ERR_CUDA; \
        }                                                                         \
    } while (0)

template <typename T>
static cudaError_t map_alloc(rtg_map_s* m, T** p, size_t count, cudaStream_t st) {
    size_t bytes = sizeof(T) * (count > 0 ? count : 1);
    cudaError_t e = dev_alloc((void**)p, bytes, st);
    if (e == cudaSuccess) {
        m->allocs.push_back(*p);
        m->bytes += (long long)bytes;
    }
    return e;
}

static void pick_dims(float lo, float hi, double h, int& n) {
    double span = (double)hi - (double)lo;
    n = (int)floor(span / h) + 1;
    if (n < 1) n = 1;
}

// Builds everything of rtg_map_create from device-resident inputs.
// grid geometry and the FP32 collision guard from bounds: the data's own (rtg_map_create) or a caller's
// layout (rtg_map_create_layout); rho bounds a_max / a_min of the collidable Gaussians
static void plan_grids(rtg_map_s* m, bool have_gain, const float glo[3], const float ghi[3], bool have_col,
                       const float clo[3], const float chi[3], double rb_max, double rho,
                       const rtg_map_options* opt) {
    m->rb_max = have_col ? (float)rb_max : 0.f;
    const double u32 = ldexp(1.0, -24);
    m->gq64 = (104.0 * (have_col ? rho : 1.0) + 6.0) * u32;   // FP32 error bound of q near 1, x2
    m->gq = (float)m->gq64;
    double hy = (opt && opt->gain_cell_xy > 0) ? opt->gain_cell_xy : 0.3;
    double hx = (opt && opt->gain_cell_x > 0) ? opt->gain_cell_x : 0.25 * hy;
    double hz = (opt && opt->gain_cell_z > 0) ? opt->gain_cell_z : 1.5;
    GainGrid& gg = m->gg;
    if (have_gain) {
        float oz = glo[2];
        for (;;) {
            pick_dims(glo[0], ghi[0], hx, gg.nx);
            pick_dims(glo[1], ghi[1], hy, gg.ny);
            if (opt && opt->gain_z_centred) {
                // z-cell boundaries at gain_z_centre +- (j + 1/2) hz: the origin moves down to the first
                // of them at or below the lowest mean (at most one more z-cell)
                const double c0 = (double)opt->gain_z_centre - 0.5 * hz;
                oz = (float)(c0 - ceil((c0 - (double)glo[2]) / hz) * hz);
                if ((double)oz > (double)glo[2]) oz = glo[2];   // (rounding: never above a mean)
            }
            pick_dims(oz, ghi[2], hz, gg.nz);
            // (the culled kernel packs cell indices in 16 bits)
            if ((double)gg.nx * gg.ny * gg.nz <= 96.0e6 && gg.nx < 65535 && gg.ny < 65535 && gg.nz < 65535) break;
            hx *= 2.0;
            hy *= 2.0;
            hz *= 2.0;
        }
        gg.ox = glo[0]; gg.oy = glo[1]; gg.oz = oz;
    } else {
        gg.nx = gg.ny = gg.nz = 1;
        gg.ox = gg.oy = gg.oz = 0.f;
    }
    gg.hx = (float)hx;
    gg.hy = (float)hy;
    gg.hz = (float)hz;
    gg.ncellsA = (long long)gg.nx * gg.ny;
    gg.nxb = (gg.nx + kZoccX - 1) / kZoccX;
    gg.ncellsB = (long long)gg.nx * gg.ny * gg.nz;
    ColGrid& cg = m->cg;
    double hc = (opt && opt->col_cell > 0) ? opt->col_cell : fmax(0.5, 0.5 * (double)m->rb_max);
    if (have_col) {
        for (;;) {
            pick_dims(clo[0], chi[0], hc, cg.nx);
            pick_dims(clo[1], chi[1], hc, cg.ny);
            pick_dims(clo[2], chi[2], hc, cg.nz);
            if ((double)cg.nx * cg.ny * cg.nz <= 64.0e6) break;
            hc *= 2.0;
        }
        cg.ox = clo[0]; cg.oy = clo[1]; cg.oz = clo[2];
    } else {
        cg.nx = cg.ny = cg.nz = 1;
        cg.ox = cg.oy = cg.oz = 0.f;
    }
    cg.h = (float)hc;
    cg.ncells = (long long)cg.nx * cg.ny * cg.nz;
}

// the map's persistent arrays for up to n_gain visibility and n_col collision records
static cudaError_t alloc_records(rtg_map_s* m, long long n_gain, long long n_col, cudaStream_t st) {
    const GainGrid& gg = m->gg;
    // >= 64 NaN records after the copy: the culled kernel's sentinel run (items past its queue)
    m->n_gain_pad = n_gain > 0 ? ((n_gain + 64 + kTile - 1) / kTile) * kTile : 0;
    m->n_col_pad = ((n_col + kTile - 1) / kTile) * kTile;
    cudaError_t e = map_alloc(m, &m->grec, 2 * m->n_gain_pad, st);
    if (e == cudaSuccess) e = map_alloc(m, &m->gidx, m->n_gain_pad, st);
    if (e == cudaSuccess) e = map_alloc(m, &m->gstartA, gg.ncellsA + 1, st);
    if (e == cudaSuccess) e = map_alloc(m, &m->zocc, (size_t)gg.ny * gg.nxb, st);
    if (e == cudaSuccess) e = map_alloc(m, &m->gtabP, (size_t)gg.ny * (gg.nx + 1) * gg.nz, st);
    if (e == cudaSuccess) e = map_alloc(m, &m->crec, m->n_col_pad, st);
    if (e == cudaSuccess) e = map_alloc(m, &m->cmat, m->n_col_pad, st);
    if (e == cudaSuccess) e = map_alloc(m, &m->csrc, m->n_col_pad, st);
    if (e == cudaSuccess) e = map_alloc(m, &m->cstart, m->cg.ncells + 1, st);
    return e;
}

// the validation pass: bounds, counts and the map's copies of the weights and flags into db
static void launch_bounds(rtg_map_s* m, long long n, const float* means, const float* quats, const float* scales,
                          const float* opacity, const float* w, const unsigned char* flags, DevBounds* db,
                          cudaStream_t st) {
    note_launch(), k_bounds_init<<<1, 1, 0, st>>>(db);
    if (n <= 0) return;
    const rtg_robot rb = m->robot;
    auto al16 = [](const void* p) { return p == nullptr || ((uintptr_t)p & 15u) == 0; };
    const bool vec = (n % 4 == 0) && al16(means) && al16(quats) && al16(scales) && al16(opacity) && al16(w) &&
                     ((uintptr_t)flags & 3u) == 0 && al16(m->w_orig) && ((uintptr_t)m->flags & 3u) == 0;
    if (vec)
        note_launch(), k_bounds<true><<<nblocks(n / 4, 256) > 1184 ? 1184 : nblocks(n / 4, 256), 256, 0, st>>>(
                           n, means, quats, scales, opacity, w, flags, rb, m->w_orig, m->flags, db);
    else
        note_launch(), k_bounds<false><<<nblocks(n, 256) > 1184 ? 1184 : nblocks(n, 256), 256, 0, st>>>(
                           n, means, quats, scales, opacity, w, flags, rb, m->w_orig, m->flags, db);
}

static rtg_status build_records(rtg_map_s* m, const float* means, const float* quats, const float* scales,
                                const float* w, const unsigned char* flags, const int* dn_gain, const int* dn_col,
                                cudaStream_t st);

// Builds everything of rtg_map_create from device-resident inputs.
rtg_status build_map(rtg_map_s* m, const float* means, const float* quats, const float* scales,
                     const float* opacity, const float* w, const unsigned char* flags, const rtg_map_options* opt,
                     cudaStream_t st) {
    long long n = m->n;
    // --- bounds + validation (one sync)
    DevBounds* db = nullptr;
    DevFreeGuard db_guard{(void**)&db, st};
    MAP_CK(dev_alloc((void**)&db, sizeof(DevBounds), st));
    // the map's own weights and flags (input order), written by the validation pass
    MAP_CK(map_alloc(m, &m->w_orig, n, st));
    if (flags) MAP_CK(map_alloc(m, &m->flags, n, st));
    // the default classification's statistics (k = 1/2, derived thresholds) depend only on
    // the inputs: they run while the host reads the bounds back, and the scatter then writes final
    // records (class increments, fixed-point u)
    MAP_CK(map_alloc(m, &m->cls, 1, st));
    MAP_CK(map_alloc(m, &m->red_scratch, 3 * kRedBlocks, st));
    launch_bounds(m, n, means, quats, scales, opacity, w, flags, db, st);
    // pinned staging (one per host thread) keeps the readback asynchronous: the classification
    // statistics below are enqueued while it is in flight
    thread_local DevBounds* hbp = nullptr;
    if (!hbp) MAP_CK(cudaMallocHost((void**)&hbp, sizeof(DevBounds)));
    DevBounds& hb = *hbp;
    MAP_CK(cudaMemcpyAsync(&hb, db, sizeof(DevBounds), cudaMemcpyDeviceToHost, st));
    cudaEvent_t ev;
    MAP_CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    MAP_CK(cudaEventRecord(ev, st));
    MAP_CK(class_stats(n, w, flags, RTG_VARIANT_XI, 0.5, NAN, NAN, m->cls, m->red_scratch, st));
    {
        cudaError_t es = cudaEventSynchronize(ev);
        cudaEventDestroy(ev);
        MAP_CK(es);
    }
    dev_free(db, st);
    db = nullptr;
    if (hb.err) {
        set_error("rtg_map_create: invalid element(s):%s%s%s%s%s", (hb.err & 1) ? " non-finite mean" : "",
                  (hb.err & 2) ? " quaternion norm < 1e-12" : "", (hb.err & 4) ? " scale <= 0 or non-finite" : "",
                  (hb.err & 8) ? " info_w < 0 or non-finite" : "", (hb.err & 16) ? " opacity outside [0,1]" : "");
        return RTG_ERR_INVALID_ARGUMENT;
    }
    m->n_gain = hb.n_gain;
    m->n_col = hb.n_col;
    float glo[3], ghi[3], clo[3], chi[3];
    for (int d = 0; d < 3; ++d) {
        glo[d] = o2f(hb.gmin[d]); ghi[d] = o2f(hb.gmax[d]);
        clo[d] = o2f(hb.cmin[d]); chi[d] = o2f(hb.cmax[d]);
    }
    plan_grids(m, m->n_gain > 0, glo, ghi, m->n_col > 0, clo, chi, m->n_col > 0 ? o2f(hb.rbmax) : 0.0,
               m->n_col > 0 ? (double)o2f(hb.rhomax) : 1.0, opt);
    MAP_CK(alloc_records(m, m->n_gain, m->n_col, st));
    return build_records(m, means, quats, scales, w, flags, nullptr, nullptr, st);
}

// the counting sorts into both grids, the record scatters, the tables (device work only).  dn_gain /
// dn_col: the record counts on the device when the host knows only upper bounds (layout maps: m->n_gain,
// m->n_col are then the capacities), else NULL and m->n_gain / m->n_col are exact.
static rtg_status build_records(rtg_map_s* m, const float* means, const float* quats, const float* scales,
                                const float* w, const unsigned char* flags, const int* dn_gain, const int* dn_col,
                                cudaStream_t st) {
    const long long n = m->n;
    const rtg_robot rb = m->robot;
    const GainGrid& gg = m->gg;
    const ColGrid& cg = m->cg;
    const double gq = m->gq64;
    // --- counting sort into both grids
    int *gkey = nullptr, *ckey = nullptr, *gcountB = nullptr, *ccount = nullptr, *gstartB = nullptr;
    // temporaries of the sort: freed (stream-ordered) on every return path
    DevFreeGuard g_gkey{(void**)&gkey, st}, g_ckey{(void**)&ckey, st}, g_gcount{(void**)&gcountB, st},
        g_gstart{(void**)&gstartB, st};
    MAP_CK(dev_alloc((void**)&gkey, sizeof(int) * (n > 0 ? n : 1), st));
    MAP_CK(dev_alloc((void**)&ckey, sizeof(int) * (n > 0 ? n : 1), st));
    int* grank = nullptr;
    int* crank = nullptr;
    DevFreeGuard g_grank{(void**)&grank, st}, g_crank{(void**)&crank, st};
    MAP_CK(dev_alloc((void**)&grank, sizeof(int) * (n > 0 ? n : 1), st));
    MAP_CK(dev_alloc((void**)&crank, sizeof(int) * (n > 0 ? n : 1), st));
    // the per-cell tables, copy A and the z-occupancy from one pass per (row, 128-column tile)
    // (k_tabs_cols) unless the grid has more than kTabsMaxZ z-cells (then: column counts and z-occupancy
    // by atomics in the key pass, the record prefix scan, k_build_tabs*, k_derive_cols_b).
    // RTG_MAP_TABLES=scan forces the latter (the parity tests compare the two).
    static const bool force_scan = getenv("RTG_MAP_TABLES") && strcmp(getenv("RTG_MAP_TABLES"), "scan") == 0;
    const bool tiles = gg.nz <= kTabsMaxZ && !force_scan;
    const int ntl = gg.nx / kTabsX + 1;   // tiles per row (the last holds the x = nx end entries)
    const long long nseg = (long long)gg.ny * gg.nz * ntl;
    // the cell-count arrays in one block, cleared by one memset (with the tile path's segment sums)
    const long long ncnt = (gg.ncellsB + 1) + (cg.ncells + 1) + (tiles ? 0 : gg.ncellsA + 1);
    const size_t cnt_bytes = (sizeof(int) * ncnt + 15) & ~(size_t)15;
    const size_t seg_bytes = tiles ? 2 * sizeof(long long) * nseg : 0;
    MAP_CK(dev_alloc((void**)&gcountB, cnt_bytes + seg_bytes, st));
    ccount = gcountB + (gg.ncellsB + 1);
    int* gcountA = tiles ? nullptr : ccount + (cg.ncells + 1);
    unsigned long long* tsum = tiles ? reinterpret_cast<unsigned long long*>((char*)gcountB + cnt_bytes) : nullptr;
    MAP_CK(dev_alloc((void**)&gstartB, sizeof(int) * (gg.ncellsB + 1), st));
    MAP_CK(cudaMemsetAsync(gcountB, 0, cnt_bytes + seg_bytes, st));
    if (!tiles)
        note_launch(), k_zocc_init<<<nblocks((long long)gg.ny * gg.nxb, 256), 256, 0, st>>>(m->zocc,
                                                                                            (long long)gg.ny * gg.nxb);
    unsigned nb = nblocks(n, 256) > 8192 ? 8192 : nblocks(n, 256);
    if (n > 0)
        note_launch(), k_keys<<<nb, 256, 0, st>>>(n, means, flags, gg, cg, gkey, ckey, grank, crank, gcountB, gcountA,
                                                  m->zocc, ccount);
    MAP_CK(cudaGetLastError());
    MAP_CK(exclusive_scan_i32(gcountB, gstartB, gg.ncellsB, st));
    MAP_CK(exclusive_scan_i32(ccount, m->cstart, cg.ncells, st));
    if (!tiles) MAP_CK(exclusive_scan_i32(gcountA, m->gstartA, gg.ncellsA, st));   // copy A's column starts
    if (n > 0) {
        // both scatters in one pass while the records they write stay near L2 size (outdoor, 136 MB:
        // 0.387 -> 0.377 ms); above, two passes (scale, 340 MB: the fused pass 17 us slower)
        const double col_bytes = (double)m->n_col * (sizeof(CRec) + sizeof(CMat) + sizeof(CSrc));
        const double gain_bytes = (double)m->n_gain * (sizeof(GRec) + sizeof(int));
        const bool scatter_gain = (double)m->n_gain * sizeof(GRec) <= kScatterMaxBytes;
        if (scatter_gain && gain_bytes + col_bytes <= kScatterBothMaxBytes) {
            note_launch(), k_scatter_both<<<nb, 256, 0, st>>>(n, means, w, quats, scales, gkey, grank, gstartB,
                                                              m->grec + m->n_gain_pad, m->gidx, RTG_VARIANT_XI,
                                                              m->cls, tsum, ntl, gg.nx, ckey, crank, m->cstart, rb,
                                                              gq, m->crec, m->cmat, m->csrc);
        } else if (scatter_gain) {
            note_launch(), k_scatter_both<<<nb, 256, 0, st>>>(n, means, w, quats, scales, gkey, grank, gstartB,
                                                              m->grec + m->n_gain_pad, m->gidx, RTG_VARIANT_XI,
                                                              m->cls, tsum, ntl, gg.nx, ckey, nullptr, m->cstart,
                                                              rb, gq, m->crec, m->cmat, m->csrc);
            note_launch(), k_scatter_col<<<nb, 256, 0, st>>>(n, means, quats, scales, ckey, crank, m->cstart, rb, gq,
                                                             m->crec, m->cmat, m->csrc);
        } else {
            GRec* rec = nullptr;
            DevFreeGuard g_rec{(void**)&rec, st};
            MAP_CK(dev_alloc((void**)&rec, sizeof(GRec) * n, st));
            note_launch(), k_pack_gain<<<nb, 256, 0, st>>>(n, means, w, rec, RTG_VARIANT_XI, m->cls);
            note_launch(), k_perm_gain<<<nb, 256, 0, st>>>(n, gkey, grank, gstartB, m->gidx, rec, tsum, ntl, gg.nx);
            const unsigned fb = nblocks(m->n_gain, 256) > 8192 ? 8192 : nblocks(m->n_gain, 256);
            note_launch(), k_fill_gain<<<fb, 256, 0, st>>>(m->n_gain, dn_gain, m->gidx, rec, m->grec + m->n_gain_pad);
            note_launch(), k_scatter_col<<<nb, 256, 0, st>>>(n, means, quats, scales, ckey, crank, m->cstart, rb, gq,
                                                             m->crec, m->cmat, m->csrc);
        }
    }
    // NaN padding after the records (a layout map: after its device counts, whatever the capacity)
    {
        const long long gfrom = dn_gain ? 0 : m->n_gain, cfrom = dn_col ? 0 : m->n_col;
        const long long span = std::max(m->n_gain_pad - gfrom, m->n_col_pad - cfrom);
        if (span > 0) {
            const unsigned pb = nblocks(span, 256) > 1184 ? 1184 : nblocks(span, 256);
            note_launch(), k_pad_records<<<pb, 256, 0, st>>>(m->grec, m->grec + m->n_gain_pad, m->gidx, gfrom,
                                                             m->n_gain_pad, dn_gain, m->crec, cfrom, m->n_col_pad,
                                                             dn_col);
        }
    }
    MAP_CK(cudaGetLastError());
    // --- default classification (k = 1/2, derived thresholds); copy A derived from copy B
    if (tiles) {
        long long* tpre = nullptr;
        DevFreeGuard g_tpre{(void**)&tpre, st};
        MAP_CK(dev_alloc((void**)&tpre, 2 * sizeof(long long) * (nseg + 1), st));
        MAP_CK(exclusive_scan_i64x2(reinterpret_cast<const long long*>(tsum), tpre, nseg, st));
        const size_t smem = tabs_smem(gg.nz);
        static bool smem_set = false;   // (> 48 KB of dynamic shared memory only for nz > 15)
        if (smem > 48 * 1024 && !smem_set) {
            MAP_CK(cudaFuncSetAttribute(k_tabs_cols, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)tabs_smem(kTabsMaxZ)));
            smem_set = true;
        }
        note_launch(), k_tabs_cols<<<dim3((unsigned)ntl, (unsigned)gg.ny), kTabsThreads, smem, st>>>(
                           gg, ntl, gstartB, reinterpret_cast<const longlong2*>(tpre), m->grec + m->n_gain_pad,
                           m->grec, m->gtabP, m->gstartA, m->zocc);
        MAP_CK(cudaGetLastError());
    } else {
        MAP_CK(class_prefix(m, st, gstartB, gcountB));
    }
    // (the guards free gkey, ckey, grank, crank, gstartB and gcountB with ccount, gcountA in its block)
    set_class_params(m, RTG_VARIANT_XI, 0.5, NAN, NAN);
    return RTG_OK;
}

// ---------------------------------------------------------------- layout maps (capturable rebuilds)

rtg_status rebuild_map(rtg_map_s* m, long long n, const float* means, const float* quats, const float* scales,
                       const float* opacity, const float* w, const unsigned char* flags, cudaStream_t st);

rtg_status create_layout_map(rtg_map_s* m, const rtg_map_layout* L, const rtg_map_options* opt, cudaStream_t st) {
    const long long cap = L->capacity;
    m->layout = true;
    m->cap = cap;
    m->lay = *L;
    m->n = 0;
    MAP_CK(map_alloc(m, &m->w_orig, cap, st));
    MAP_CK(map_alloc(m, &m->flags, cap, st));
    MAP_CK(map_alloc(m, &m->cls, 1, st));
    MAP_CK(map_alloc(m, &m->red_scratch, 3 * kRedBlocks, st));
    DevBounds* db = nullptr;
    MAP_CK(map_alloc(m, &db, 1, st));
    m->dbounds = db;
    plan_grids(m, true, L->gain_lo, L->gain_hi, true, L->col_lo, L->col_hi, L->rb_max, L->rho_max, opt);
    MAP_CK(alloc_records(m, cap, cap, st));
    // an empty map until the first rebuild (every array written)
    return rebuild_map(m, 0, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, st);
}

rtg_status rebuild_map(rtg_map_s* m, long long n, const float* means, const float* quats, const float* scales,
                       const float* opacity, const float* w, const unsigned char* flags, cudaStream_t st) {
    DevBounds* db = static_cast<DevBounds*>(m->dbounds);
    m->n = n;
    m->n_gain = m->n_col = m->cap;   // upper bounds until rtg_map_check reads the counts
    if (!flags && n > 0) MAP_CK(cudaMemsetAsync(m->flags, 0, (size_t)n, st));
    launch_bounds(m, n, means, quats, scales, opacity, w, flags, db, st);
    note_launch(), k_layout_check<<<1, 32, 0, st>>>(db, m->lay);
    MAP_CK(class_stats(n, m->w_orig, m->flags, RTG_VARIANT_XI, 0.5, NAN, NAN, m->cls, m->red_scratch, st));
    set_class_params(m, RTG_VARIANT_XI, 0.5, NAN, NAN);
    return build_records(m, means, quats, scales, m->w_orig, m->flags, &db->n_gain, &db->n_col, st);
}

rtg_status check_layout_map(rtg_map_s* m, cudaStream_t st) {
    DevBounds hb;
    MAP_CK(cudaMemcpyAsync(&hb, m->dbounds, sizeof(DevBounds), cudaMemcpyDeviceToHost, st));
    MAP_CK(cudaStreamSynchronize(st));
    if (hb.err) {
        set_error("rtg_map_check: the last rebuild's data is invalid:%s%s%s%s%s%s%s%s%s",
                  (hb.err & 1) ? " non-finite mean" : "", (hb.err & 2) ? " quaternion norm < 1e-12" : "",
                  (hb.err & 4) ? " scale <= 0 or non-finite" : "", (hb.err & 8) ? " info_w < 0 or non-finite" : "",
                  (hb.err & 16) ? " opacity outside [0,1]" : "",
                  (hb.err & 32) ? " gain-eligible mean outside the layout box" : "",
                  (hb.err & 64) ? " collidable mean outside the layout box" : "",
                  (hb.err & 128) ? " semi-axis above rb_max" : "", (hb.err & 256) ? " anisotropy above rho_max" : "");
        return RTG_ERR_INVALID_ARGUMENT;
    }
    m->n_gain = hb.n_gain;
    m->n_col = hb.n_col;
    return RTG_OK;
}

}  // namespace rtg
