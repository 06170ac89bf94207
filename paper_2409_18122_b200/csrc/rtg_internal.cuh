// rtg_internal.cuh -- shared device-side definitions of librtg (sm_100a).
//
// The pair tests live here ONCE and are used by both execution modes (dense and
// culled) and the debug kernels, so every mode takes identical decisions.
//
// Numerics:
//  * collision:  q32 = sum_i (M_i . d)^2 in FP32 with M = diag(1/a) R^T packed in FP64 and
//    rounded once (SURVEY F2 / [A2], [A11]); pairs with |q32 - 1| < gq are re-decided in
//    FP64 from the FP64-packed M (same formula as the oracle, O2).
//  * visibility: min slack m32 of the folded frustum (|Z - zmid| <= zhalf,
//    |X - kxc Z| <= kxh Z, |dz - kyc Z| <= kyh Z); pairs with |m32| < gam*Z + g0 are
//    re-decided in FP64 with the six pinhole slacks (O3).  gam, g0 bound the FP32 error.
//  * gains: u_q = round(u * 2^S) < 2^30 with S chosen so that the sum over ALL eligible Gaussians
//    is < 2^53: every partial sum is an exact integer in FP64 (associative -> order free).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/rtg.h"

namespace rtg {

constexpr int kTile = 512;           // dense-mode Gaussians per smem tile
constexpr int kZoccX = 64;           // x-cells per block of the visibility grid's z-occupancy table

// ------------------------------------------------------------------ records
// visibility record (sorted by visibility cell): mean + uc = u_q | c << 24 with u_q the
// fixed-point u (< 2^24, exact integer) and the class byte c = kClsH (H), kClsL (L), 0 (O): a
// per-lane 32-bit sum of up to 127 words still separates sum(u_q) and nH + 128 nL (culled kernel)
struct __align__(16) GRec { float x, y, z; unsigned uc; };
constexpr int kUqBits = 24;
constexpr unsigned kUqMask = (1u << kUqBits) - 1u;
constexpr unsigned kClsH = 1u, kClsL = 0x80u;
// per-lane packed class counter increment of uc: 1 (H), 0x10000 (L), 0 (O)
__device__ __forceinline__ int uc_inc(unsigned uc) {
    const unsigned c = uc >> kUqBits;
    return (int)((c & kClsH) | ((c & kClsL) << 9));
}
// collision record (sorted by collision cell): mean + inflated bounding radius^2
struct __align__(16) CRec { float x, y, z, rb2; };
// M rows (FP32): m[0..8] row-major, m[9] = original index (as int bits), pad
struct __align__(16) CMat { float m[12]; };
// z-fastest table entry at a copy-B cell boundary: the cell's first record and the exact exclusive
// prefixes there, packed modulo 2^48 (sum of u_q) and 2^24 (class counts nH, nL):
// {start, q[31:0], q[47:32] | nH[15:0] << 16, nH[23:16] | nL << 8}
struct __align__(16) TabP { int start; unsigned qlo, qhi_nh, nh_nl; };
// the fp32 inputs M is packed from (sorted like the collision records): the rare FP64
// re-decision recomputes M from them with the same code as the packing (pack_m64)
struct __align__(32) CSrc { float q[4]; float s[3]; float pad; };

// a1 in FP64: inflated semi-axes a_i = lambda_g s_i + r_robot (PRINCIPAL_AXIS: every
// a_i = lambda_g max s + r_robot) and M = diag(1/a) R^T with R the Hamilton rotation of
// the normalised quaternion (w, x, y, z).  Used for packing and for every FP64 re-decision.
__device__ __forceinline__ void semi_axes64(double s0, double s1, double s2, const rtg_robot& rb, double a[3]) {
    if (rb.collide_rule == RTG_COLLIDE_PRINCIPAL_AXIS) {
        const double r = (double)rb.lambda_g * fmax(s0, fmax(s1, s2)) + (double)rb.r_robot;
        a[0] = a[1] = a[2] = r;
        return;
    }
    a[0] = (double)rb.lambda_g * s0 + (double)rb.r_robot;
    a[1] = (double)rb.lambda_g * s1 + (double)rb.r_robot;
    a[2] = (double)rb.lambda_g * s2 + (double)rb.r_robot;
}

__device__ __forceinline__ void pack_m64(double qw, double qx, double qy, double qz, double s0, double s1, double s2,
                                         const rtg_robot& rb, double M[9], double a[3]) {
    semi_axes64(s0, s1, s2, rb, a);
    if (rb.collide_rule == RTG_COLLIDE_PRINCIPAL_AXIS) {
        for (int j = 0; j < 9; ++j) M[j] = 0.0;
        M[0] = M[4] = M[8] = 1.0 / a[0];
        return;
    }
    const double nq = sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
    qw /= nq; qx /= nq; qy /= nq; qz /= nq;
    // Hamilton R (columns = local principal axes)
    const double R[3][3] = {
        {1.0 - 2.0 * (qy * qy + qz * qz), 2.0 * (qx * qy - qw * qz), 2.0 * (qx * qz + qw * qy)},
        {2.0 * (qx * qy + qw * qz), 1.0 - 2.0 * (qx * qx + qz * qz), 2.0 * (qy * qz - qw * qx)},
        {2.0 * (qx * qz - qw * qy), 2.0 * (qy * qz + qw * qx), 1.0 - 2.0 * (qx * qx + qy * qy)}};
    for (int r = 0; r < 3; ++r)         // row r of M = column r of R / a_r  (M = diag(1/a) R^T)
        for (int c = 0; c < 3; ++c) M[3 * r + c] = R[c][r] / a[r];
}

// ------------------------------------------------------------------ camera constants
struct CamK {
    float zmid, zhalf;   // depth  |Z - zmid| <= zhalf
    float kxc, kxh;      // horiz  |X - kxc Z| <= kxh Z
    float kyc, kyh;      // vert   |dz - kyc Z| <= kyh Z
    float gam, g0;       // FP32 guard: FP64 re-decision iff |m32| < gam*Z + g0
    const double* cam64; // device: {W, H, fx, fy, cx, cy, z_near, z_far} for the FP64 slacks
};

// per-waypoint constants (yaw kept for the rare FP64 re-decision)
struct WpF { float px, py, pz, c, s, ax, bx, yaw; };

__device__ __forceinline__ void wp_setup_cs(float x, float y, float z, float yaw, const CamK& k, WpF& f,
                                            double& cs, double& sn) {
    sincos((double)yaw, &sn, &cs);
    f.px = x; f.py = y; f.pz = z; f.yaw = yaw;
    f.c = (float)cs; f.s = (float)sn;
    f.ax = (float)(sn - (double)k.kxc * cs);
    f.bx = (float)(-cs - (double)k.kxc * sn);
}

// same, from a precomputed FP64 (cos, sin) of the yaw
__device__ __forceinline__ void wp_setup_from_cs(float x, float y, float z, float yaw, double cs, double sn,
                                                 const CamK& k, WpF& f) {
    f.px = x; f.py = y; f.pz = z; f.yaw = yaw;
    f.c = (float)cs; f.s = (float)sn;
    f.ax = (float)(sn - (double)k.kxc * cs);
    f.bx = (float)(-cs - (double)k.kxc * sn);
}

__device__ __forceinline__ void wp_setup(float x, float y, float z, float yaw, const CamK& k, WpF& f) {
    double sn, cs;
    sincos((double)yaw, &sn, &cs);
    f.px = x; f.py = y; f.pz = z; f.yaw = yaw;
    f.c = (float)cs; f.s = (float)sn;
    // X' = X - kxc Z with X = s dx - c dy, Z = c dx + s dy  (coefficients rounded once)
    f.ax = (float)(sn - (double)k.kxc * cs);
    f.bx = (float)(-cs - (double)k.kxc * sn);
}

// ------------------------------------------------------------------ visibility
// FP32 margin: min over the three folded slack pairs (>= 0 <=> visible in FP32)
__device__ __forceinline__ float vis_margin(const WpF& w, const CamK& k, float mx, float my,
                                            float mz, float& Z) {
    float dx = mx - w.px, dy = my - w.py, dz = mz - w.pz;
    Z = fmaf(w.c, dx, w.s * dy);
    float X = fmaf(w.ax, dx, w.bx * dy);
    float Y = fmaf(-k.kyc, Z, dz);
    float s1 = k.zhalf - fabsf(Z - k.zmid);
    float s2 = fmaf(k.kxh, Z, -fabsf(X));
    float s3 = fmaf(k.kyh, Z, -fabsf(Y));
    return fminf(s1, fminf(s2, s3));
}

// Blackwell's packed FP32 (f32x2: FADD2 / FMUL2 / FFMA2 on register pairs, scalar operands
// broadcast): each half rounds exactly like the scalar instruction.
__device__ __forceinline__ unsigned long long f2_pack(float lo, float hi) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void f2_unpack(unsigned long long v, float& lo, float& hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ unsigned long long f2_add(unsigned long long a, unsigned long long b) {
    unsigned long long d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ unsigned long long f2_sub(unsigned long long a, unsigned long long b) {
    unsigned long long d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ unsigned long long f2_mul(unsigned long long a, unsigned long long b) {
    unsigned long long d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ unsigned long long f2_fma(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
// one item with the packed pairs (x, y) and (Z, X') of the same Gaussian, so the record's own
// register pair feeds the first FADD2 (no re-pairing moves); rounds exactly like vis_margin
// Also returns the FP32 guard gam Z + g0.
__device__ __forceinline__ float vis_margin_xy(const WpF& w, const CamK& k, float mx, float my, float mz,
                                               float& guard) {
    float dx, dy, Z, X;
    f2_unpack(f2_sub(f2_pack(mx, my), f2_pack(w.px, w.py)), dx, dy);
    f2_unpack(f2_fma(f2_pack(w.c, w.ax), f2_pack(dx, dx), f2_mul(f2_pack(w.s, w.bx), f2_pack(dy, dy))), Z, X);
    const float Y = fmaf(-k.kyc, Z, mz - w.pz);
    guard = fmaf(k.gam, Z, k.g0);
    return fminf(k.zhalf - fabsf(Z - k.zmid), fminf(fmaf(k.kxh, Z, -fabsf(X)), fmaf(k.kyh, Z, -fabsf(Y))));
}

// two waypoints against one item (dense mode): the waypoints' constants as register pairs, the
// item broadcast; each half rounds exactly like vis_margin (bit-identical margins)
struct WpF2 {
    unsigned long long px, py, pz, c, s, ax, bx;
};
__device__ __forceinline__ WpF2 wp_pair(const WpF& a, const WpF& b) {
    return WpF2{f2_pack(a.px, b.px), f2_pack(a.py, b.py), f2_pack(a.pz, b.pz), f2_pack(a.c, b.c),
                f2_pack(a.s, b.s),   f2_pack(a.ax, b.ax), f2_pack(a.bx, b.bx)};
}
__device__ __forceinline__ void vis_margin_w2(const WpF2& w, const CamK& k, float mx, float my, float mz, float& ma,
                                              float& mb, float& ga, float& gb) {
    const unsigned long long dx = f2_sub(f2_pack(mx, mx), w.px);
    const unsigned long long dy = f2_sub(f2_pack(my, my), w.py);
    const unsigned long long dz = f2_sub(f2_pack(mz, mz), w.pz);
    const unsigned long long Z = f2_fma(w.c, dx, f2_mul(w.s, dy));
    const unsigned long long X = f2_fma(w.ax, dx, f2_mul(w.bx, dy));
    const unsigned long long Y = f2_fma(f2_pack(-k.kyc, -k.kyc), Z, dz);
    const unsigned long long D = f2_sub(Z, f2_pack(k.zmid, k.zmid));
    const unsigned long long G = f2_fma(f2_pack(k.gam, k.gam), Z, f2_pack(k.g0, k.g0));
    float Za, Zb, Xa, Xb, Ya, Yb, Da, Db;
    f2_unpack(Z, Za, Zb);
    f2_unpack(X, Xa, Xb);
    f2_unpack(Y, Ya, Yb);
    f2_unpack(D, Da, Db);
    f2_unpack(G, ga, gb);
    ma = fminf(k.zhalf - fabsf(Da), fminf(fmaf(k.kxh, Za, -fabsf(Xa)), fmaf(k.kyh, Za, -fabsf(Ya))));
    mb = fminf(k.zhalf - fabsf(Db), fminf(fmaf(k.kxh, Zb, -fabsf(Xb)), fmaf(k.kyh, Zb, -fabsf(Yb))));
}

// FP64 decision with the six slacks of the pinhole test (visible <=> all >= 0), cos/sin of the
// yaw given in FP64.  Every product is an explicit fma/mul so all kernels round identically.
__device__ __forceinline__ bool vis_decide64_cs(float px, float py, float pz, double cs, double sn, float mx,
                                                float my, float mz, const double* __restrict__ k) {
    const double W = __ldg(k + 0), H = __ldg(k + 1), fx = __ldg(k + 2), fy = __ldg(k + 3);
    const double cx = __ldg(k + 4), cy = __ldg(k + 5), zn = __ldg(k + 6), zf = __ldg(k + 7);
    const double dx = (double)mx - (double)px, dy = (double)my - (double)py, dz = (double)mz - (double)pz;
    const double Z = fma(cs, dx, sn * dy);
    const double X = fma(sn, dx, -(cs * dy));
    const double Y = -dz;
    bool v = (Z - zn >= 0.0) & (zf - Z >= 0.0);
    v &= (fma(fx, X, cx * Z) >= 0.0) & (fma(W - cx, Z, -(fx * X)) >= 0.0);
    v &= (fma(fy, Y, cy * Z) >= 0.0) & (fma(H - cy, Z, -(fy * Y)) >= 0.0);
    return v;
}

// same decision recomputing cos/sin (dense kernels keep no FP64 registers per waypoint); rare path
static __device__ __noinline__ bool vis_decide64(float px, float py, float pz, float yaw, float mx, float my, float mz,
                                                 const double* __restrict__ k) {
    double sn, cs;
    sincos((double)yaw, &sn, &cs);
    return vis_decide64_cs(px, py, pz, cs, sn, mx, my, mz, k);
}

// exact-decision visibility of one pair; `nref` counts FP64 re-decisions
__device__ __forceinline__ bool visible(const WpF& w, const CamK& k, float mx, float my, float mz,
                                        unsigned& nref) {
    float Z;
    float m = vis_margin(w, k, mx, my, mz, Z);
    bool v = m >= 0.0f;
    if (fabsf(m) < fmaf(k.gam, Z, k.g0)) {
        v = vis_decide64(w.px, w.py, w.pz, w.yaw, mx, my, mz, k.cam64);
        ++nref;
    }
    return v;
}

// same, with the waypoint's FP64 cos/sin at hand (culled kernel: kept in shared memory)
__device__ __forceinline__ bool visible_cs(const WpF& w, const CamK& k, float mx, float my, float mz,
                                           const double* cs_sn, unsigned& nref) {
    float Z;
    float m = vis_margin(w, k, mx, my, mz, Z);
    bool v = m >= 0.0f;
    if (fabsf(m) < fmaf(k.gam, Z, k.g0)) {
        v = vis_decide64_cs(w.px, w.py, w.pz, cs_sn[0], cs_sn[1], mx, my, mz, k.cam64);
        ++nref;
    }
    return v;
}

// ------------------------------------------------------------------ collision
static __device__ __noinline__ bool col_decide64(const CSrc* __restrict__ src, const rtg_robot rb, float px, float py,
                                                 float pz, float mx, float my, float mz) {
    const CSrc c = *src;
    double M[9], a[3];
    pack_m64(c.q[0], c.q[1], c.q[2], c.q[3], c.s[0], c.s[1], c.s[2], rb, M, a);
    double dx = (double)px - (double)mx, dy = (double)py - (double)my, dz = (double)pz - (double)mz;
    double e0 = M[0] * dx + M[1] * dy + M[2] * dz;
    double e1 = M[3] * dx + M[4] * dy + M[5] * dz;
    double e2 = M[6] * dx + M[7] * dy + M[8] * dz;
    return e0 * e0 + e1 * e1 + e2 * e2 < 1.0;
}

// full quadratic form for a sphere-passing pair
__device__ __forceinline__ bool collide_full(const float* m, float dx, float dy, float dz, float gq,
                                             const CSrc* src, const rtg_robot& rb, float px, float py, float pz,
                                             float mx, float my, float mz, unsigned& nref) {
    float e0 = fmaf(m[0], dx, fmaf(m[1], dy, m[2] * dz));
    float e1 = fmaf(m[3], dx, fmaf(m[4], dy, m[5] * dz));
    float e2 = fmaf(m[6], dx, fmaf(m[7], dy, m[8] * dz));
    float q = fmaf(e0, e0, fmaf(e1, e1, e2 * e2));
    bool c = q < 1.0f;
    if (fabsf(q - 1.0f) < gq) {
        c = col_decide64(src, rb, px, py, pz, mx, my, mz);
        ++nref;
    }
    return c;
}


// ------------------------------------------------------------------ culled collision of one point
struct ColGridK {
    float ox, oy, oz, h, R;   // collision grid origin, cell edge, stencil radius (>= every r_b)
    int nx, ny, nz;
};

__device__ __forceinline__ int clamp_cell(float v, int lo, int hi) {
    v = fminf(fmaxf(v, (float)lo - 1.0f), (float)hi + 1.0f);
    int c = (int)floorf(v);
    return c;
}

// Warp-cooperative exact collision test of point p against the collidable Gaussians (a4, O2):
// the cell rows of the +-R box are flattened over the lanes, each candidate gets the sphere reject
// and, when it passes, the full quadratic form (FP32 + FP64 re-decision in the guard band); stops
// at the first collision.  Every lane returns the result.  A NaN point collides with nothing.
__device__ __forceinline__ bool warp_point_collides(float px, float py, float pz, const CRec* __restrict__ crec,
                                                    const CMat* __restrict__ cmat, const CSrc* __restrict__ csrc,
                                                    const rtg_robot& rb, const int* __restrict__ cstart,
                                                    const ColGridK& g, float gq, unsigned& nref,
                                                    unsigned long long& ntest) {
    constexpr unsigned kAll = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    bool hit = false;
    if (!(isfinite(px) && isfinite(py) && isfinite(pz))) return false;
    int ix0 = max(0, clamp_cell((px - g.R - g.ox) / g.h, 0, g.nx));
    int ix1 = min(g.nx - 1, clamp_cell((px + g.R - g.ox) / g.h, 0, g.nx));
    int iy0 = max(0, clamp_cell((py - g.R - g.oy) / g.h, 0, g.ny));
    int iy1 = min(g.ny - 1, clamp_cell((py + g.R - g.oy) / g.h, 0, g.ny));
    int iz0 = max(0, clamp_cell((pz - g.R - g.oz) / g.h, 0, g.nz));
    int iz1 = min(g.nz - 1, clamp_cell((pz + g.R - g.oz) / g.h, 0, g.nz));
    if (ix0 > ix1 || iy0 > iy1 || iz0 > iz1) return false;
    const int nyr = iy1 - iy0 + 1;
    const int nrows = nyr * (iz1 - iz0 + 1);
    for (int r0 = 0; r0 < nrows && !hit; r0 += 32) {
        const int r = r0 + lane;
        int beg = 0, len = 0;
        if (r < nrows) {
            int iz = iz0 + r / nyr, iy = iy0 + r % nyr;
            long long base = ((long long)iz * g.ny + iy) * g.nx;
            beg = cstart[base + ix0];
            len = cstart[base + ix1 + 1] - beg;
        }
        int incl = len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int v = __shfl_up_sync(kAll, incl, o);
            if (lane >= o) incl += v;
        }
        const int total = __shfl_sync(kAll, incl, 31);
        const int roff = beg - (incl - len);
        for (int b0 = 0; b0 < total; b0 += 32) {
            const int pos = b0 + lane;
            // row owning candidate pos: first lane whose inclusive prefix exceeds it
            int owner = 0;
#pragma unroll
            for (int st = 16; st > 0; st >>= 1) {
                const int v = __shfl_sync(kAll, incl, owner + st - 1);
                if (v <= pos) owner += st;
            }
            const int gi = pos + __shfl_sync(kAll, roff, owner);
            bool h = false;
            if (pos < total) {
                const CRec A = crec[gi];
                float dx = px - A.x, dy = py - A.y, dz = pz - A.z;
                float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
                if (d2 < A.rb2)
                    h = collide_full(cmat[gi].m, dx, dy, dz, gq, &csrc[gi], rb, px, py, pz, A.x, A.y, A.z, nref);
            }
            ntest += (unsigned long long)min(32, total - b0);
            if (__any_sync(kAll, h)) {
                hit = true;
                break;
            }
        }
        __syncwarp();
    }
    return hit;
}

constexpr int kUnionFactor = 3;

// the points of `live` (lanes) one at a time, ascending (the first hit is the lowest point); out of line,
// so the common union-box path keeps its registers
static __device__ __noinline__ unsigned warp_points_collide_each(float px, float py, float pz, unsigned live,
                                                                 bool first_only, const CRec* __restrict__ crec,
                                                                 const CMat* __restrict__ cmat,
                                                                 const CSrc* __restrict__ csrc, const rtg_robot rb,
                                                                 const int* __restrict__ cstart, const ColGridK g,
                                                                 float gq, unsigned& nref, unsigned long long& ntest) {
    constexpr unsigned kAll = 0xffffffffu;
    unsigned hits = 0u;
    for (unsigned lv = live; lv; lv &= lv - 1) {
        const int jj = __ffs(lv) - 1;
        const float qx = __shfl_sync(kAll, px, jj), qy = __shfl_sync(kAll, py, jj), qz = __shfl_sync(kAll, pz, jj);
        if (warp_point_collides(qx, qy, qz, crec, cmat, csrc, rb, cstart, g, gq, nref, ntest)) {
            hits |= 1u << jj;
            if (first_only) break;
        }
    }
    return hits;
}

// which of the nj points held by lanes 0 .. nj-1 collide (bit j: lane j's point; warp-uniform)?
// The candidates of the union of their cell boxes are loaded once and each is tested against every
// point: a Gaussian outside a point's own box lies beyond g.R, past its bounding radius, so the sphere
// test rejects it for that point and every decision equals the one-point test above.  Points at or
// past the lowest colliding one are skipped when only the first collision matters (first_only).
__device__ __forceinline__ unsigned warp_points_collide_mask(float px, float py, float pz, int nj, bool first_only,
                                                             const CRec* __restrict__ crec,
                                                             const CMat* __restrict__ cmat,
                                                             const CSrc* __restrict__ csrc, const rtg_robot& rb,
                                                             const int* __restrict__ cstart, const ColGridK& g,
                                                             float gq, unsigned& nref, unsigned long long& ntest) {
    constexpr unsigned kAll = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const bool mine = lane < nj && isfinite(px) && isfinite(py) && isfinite(pz);
    int ix0 = INT_MAX, ix1 = -1, iy0 = INT_MAX, iy1 = -1, iz0 = INT_MAX, iz1 = -1;
    if (mine) {
        const int a0 = max(0, clamp_cell((px - g.R - g.ox) / g.h, 0, g.nx));
        const int a1 = min(g.nx - 1, clamp_cell((px + g.R - g.ox) / g.h, 0, g.nx));
        const int b0 = max(0, clamp_cell((py - g.R - g.oy) / g.h, 0, g.ny));
        const int b1 = min(g.ny - 1, clamp_cell((py + g.R - g.oy) / g.h, 0, g.ny));
        const int c0 = max(0, clamp_cell((pz - g.R - g.oz) / g.h, 0, g.nz));
        const int c1 = min(g.nz - 1, clamp_cell((pz + g.R - g.oz) / g.h, 0, g.nz));
        if (a0 <= a1 && b0 <= b1 && c0 <= c1) {
            ix0 = a0; ix1 = a1; iy0 = b0; iy1 = b1; iz0 = c0; iz1 = c1;
        }
    }
    const unsigned live = __ballot_sync(kAll, ix0 <= ix1);
    if (!live) return 0u;
    // the union box grows with the square (cube) of the points' spread: sparse or diagonal waypoints
    // (1 s primitives, user trajectories) would load far more candidates than their own boxes hold.
    // Above kUnionFactor x the sum of the per-point boxes, test the points one at a time instead.
    const unsigned own = ix0 <= ix1 ? (unsigned)((ix1 - ix0 + 1) * (iy1 - iy0 + 1) * (iz1 - iz0 + 1)) : 0u;
    const unsigned own_sum = __reduce_add_sync(kAll, own);
    ix0 = __reduce_min_sync(kAll, ix0);
    ix1 = __reduce_max_sync(kAll, ix1);
    iy0 = __reduce_min_sync(kAll, iy0);
    iy1 = __reduce_max_sync(kAll, iy1);
    iz0 = __reduce_min_sync(kAll, iz0);
    iz1 = __reduce_max_sync(kAll, iz1);
    if ((long long)(ix1 - ix0 + 1) * (iy1 - iy0 + 1) * (iz1 - iz0 + 1) > (long long)kUnionFactor * own_sum)
        return warp_points_collide_each(px, py, pz, live, first_only, crec, cmat, csrc, rb, cstart, g, gq, nref, ntest);
    const int nyr = iy1 - iy0 + 1;
    const int nrows = nyr * (iz1 - iz0 + 1);
    unsigned hits = 0u, todo = live;
    for (int r0 = 0; r0 < nrows && todo; r0 += 32) {
        const int r = r0 + lane;
        int beg = 0, len = 0;
        if (r < nrows) {
            const int iz = iz0 + r / nyr, iy = iy0 + r % nyr;
            const long long base = ((long long)iz * g.ny + iy) * g.nx;
            beg = cstart[base + ix0];
            len = cstart[base + ix1 + 1] - beg;
        }
        int incl = len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(kAll, incl, o);
            if (lane >= o) incl += v;
        }
        const int total = __shfl_sync(kAll, incl, 31);
        const int roff = beg - (incl - len);
        for (int b0 = 0; b0 < total && todo; b0 += 32) {
            const int pos = b0 + lane;
            int owner = 0;
#pragma unroll
            for (int st = 16; st > 0; st >>= 1) {
                const int v = __shfl_sync(kAll, incl, owner + st - 1);
                if (v <= pos) owner += st;
            }
            const int gi = pos + __shfl_sync(kAll, roff, owner);
            CRec A;
            if (pos < total) A = crec[gi];
            unsigned mh = 0u;
            for (unsigned lv = todo; lv; lv &= lv - 1) {   // warp-uniform loop over the open points
                const int jj = __ffs(lv) - 1;
                const float qx = __shfl_sync(kAll, px, jj), qy = __shfl_sync(kAll, py, jj),
                            qz = __shfl_sync(kAll, pz, jj);
                if (pos < total) {
                    const float dx = qx - A.x, dy = qy - A.y, dz = qz - A.z;
                    const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
                    if (d2 < A.rb2 && collide_full(cmat[gi].m, dx, dy, dz, gq, &csrc[gi], rb, qx, qy, qz, A.x, A.y,
                                                   A.z, nref))
                        mh |= 1u << jj;
                }
            }
            ntest += (unsigned long long)min(32, total - b0) * __popc(todo);
            mh = __reduce_or_sync(kAll, mh);
            hits |= mh;
            todo &= ~mh;
            if (first_only && hits) todo &= (1u << (__ffs(hits) - 1)) - 1u;   // only earlier points matter
        }
        __syncwarp();
    }
    return hits;
}

// ------------------------------------------------------------------ misc helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// TMA 1-D bulk copy global -> shared, completion tracked by an mbarrier (sm_90+; UBLKCP in SASS)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

}  // namespace rtg
