// rtg_gain_culled.cu -- exact culled visibility + information gain.
//
// One warp per info waypoint (persistent warps pull waypoints from an atomic counter in
// (k, t) order, so neighbouring warps share frusta and L1/L2 lines).  Per waypoint:
//   1. the frustum's xy footprint is the trapezoid {z_near <= Z <= z_far, -kxl Z <= X <= kxr Z};
//      lanes take the visibility-grid rows it covers and clip the trapezoid to each row band;
//   2. lanes take the covered columns (load-balanced over rows).  A column's square is tested
//      against the linear horizontal constraints (centre +- radius); for a column entirely
//      inside, the z-cells whose whole height is inside the vertical wedge at the column's
//      smallest depth are summed from the exact fixed-point prefix records (two loads), the
//      z-cells the wedge may cut form at most two contiguous record runs; a straddling column
//      contributes one run (its candidate z-range);
//   3. the runs' Gaussians are tested one by one with the shared exact pair test (FP32 +
//      FP64 re-decision), lanes load-balanced over the union of the runs.
// All sums are integers (fixed-point u, packed class counts): exact and order free, so the
// result is bit-identical to the dense kernel.
#include <cfloat>

#include "rtg_host.hpp"

namespace rtg {
namespace {

constexpr unsigned kFullG = 0xffffffffu;
constexpr int kWarpsG = 8;

struct GainK {
    float ox, oy, oz, h, hz, hh, eps, inv_h, inv_hz;
    int nx, ny, nz;
    float zn, zf, kxl, kxr, kyu, kyd, kxh;
};

constexpr int kLongRun = 16;   // runs at least this long are tested run by run, whole warp

// acc += q and pc += inc when p (predicated adds, no selects)
__device__ __forceinline__ void add_if(bool p, long long& acc, long long q, int& pc, int inc) {
    asm("{\n\t.reg .pred pp;\n\tsetp.ne.b32 pp, %4, 0;\n\t@pp add.s64 %0, %0, %2;\n\t@pp add.s32 %1, %1, %3;\n\t}"
        : "+l"(acc), "+r"(pc)
        : "l"(q), "r"(inc), "r"((int)p));
}

__device__ __forceinline__ int fcell(float v, int hi) {   // floor of v clamped to [-1, hi + 1]
    v = fminf(fmaxf(v, -1.0f), (float)hi + 1.0f);
    return (int)floorf(v);
}

template <bool kStats>
__global__ void __launch_bounds__(kWarpsG * 32, 4) k_gain_culled(
    const float* __restrict__ X, const float* __restrict__ Y, const float* __restrict__ Zw,
    const float* __restrict__ Yaw, const int* __restrict__ list, const int* __restrict__ list_count,
    const GRec* __restrict__ grec, const long long* __restrict__ guq, const int* __restrict__ gstart,
    const CellAgg* __restrict__ agg, const GainK g, const CamK cam,
    long long* __restrict__ wp_gq, int* __restrict__ wp_nh, int* __restrict__ wp_nl, int* __restrict__ counter,
    unsigned long long* __restrict__ stats) {
    __shared__ double s_cs[kWarpsG][2];     // FP64 cos, sin of the waypoint's yaw (re-decisions)
    __shared__ float s_k[kWarpsG][8];       // per-waypoint column-test constants
    __shared__ float s_v[kWarpsG][8];       // footprint vertices (x0..x3, y0..y3)
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int L = *list_count;
    unsigned nref = 0;
    unsigned long long ntest = 0, nagg = 0, ncol = 0, nstr = 0, nvis = 0;
    for (;;) {
        int e = 0;
        if (lane == 0) e = atomicAdd(counter, 1);
        e = __shfl_sync(kFullG, e, 0);
        if (e >= L) break;
        const int i = list[e];
        const float px = X[i], py = Y[i], pz = Zw[i], yw = Yaw[i];
        long long accq = 0;
        int acch = 0, accl = 0;
        if (isfinite(px) && isfinite(py) && isfinite(pz) && isfinite(yw)) {
            WpF f;
            {
                double cs, sn;
                wp_setup_cs(px, py, pz, yw, cam, f, cs, sn);
                const float qx = px - g.ox, qy = py - g.oy;
                if (lane < 4) {     // vertex = p + Z (c, s) + kZ (s, -c)
                    const float zz = lane < 2 ? g.zn : g.zf;
                    const float kk = (lane == 0 || lane == 3) ? -g.kxl : g.kxr;
                    s_v[wid][lane] = fmaf(zz, fmaf(kk, f.s, f.c), qx);
                    s_v[wid][4 + lane] = fmaf(zz, fmaf(-kk, f.c, f.s), qy);
                }
                if (lane == 0) {
                    s_cs[wid][0] = cs;
                    s_cs[wid][1] = sn;
                    // column-test radii of the linear functions Z, kxh Z -+ X' over an h x h square
                    s_k[wid][0] = (fabsf(f.c) + fabsf(f.s)) * g.hh;
                    s_k[wid][1] = (fabsf(fmaf(g.kxh, f.c, -f.ax)) + fabsf(fmaf(g.kxh, f.s, -f.bx))) * g.hh;
                    s_k[wid][2] = (fabsf(fmaf(g.kxh, f.c, f.ax)) + fabsf(fmaf(g.kxh, f.s, f.bx))) * g.hh;
                    s_k[wid][3] = qx;
                    s_k[wid][4] = qy;
                    s_k[wid][5] = pz - g.oz;
                }
                __syncwarp();
            }
            const float ymn = fminf(fminf(s_v[wid][4], s_v[wid][5]), fminf(s_v[wid][6], s_v[wid][7])) - g.eps;
            const float ymx = fmaxf(fmaxf(s_v[wid][4], s_v[wid][5]), fmaxf(s_v[wid][6], s_v[wid][7])) + g.eps;
            const int iy0 = max(0, fcell(ymn * g.inv_h, g.ny));
            const int iy1 = min(g.ny - 1, fcell(ymx * g.inv_h, g.ny));
            for (int rbase = iy0; rbase <= iy1; rbase += 32) {
                const int iy = rbase + lane;
                int ixlo = 0, len = 0;
                if (iy <= iy1) {
                    const float yb0 = iy * g.h - g.eps, yb1 = (iy + 1) * g.h + g.eps;
                    float xlo = FLT_MAX, xhi = -FLT_MAX;
#pragma unroll
                    for (int ed = 0; ed < 4; ++ed) {
                        const float ax = s_v[wid][ed], ay = s_v[wid][4 + ed];
                        const float bx = s_v[wid][(ed + 1) & 3], by = s_v[wid][4 + ((ed + 1) & 3)];
                        const float elo = fminf(ay, by), ehi = fmaxf(ay, by);
                        if (ehi < yb0 || elo > yb1) continue;
                        float xa = ax, xb = bx;
                        if (ehi - elo > 1e-12f) {
                            const float inv = __fdividef(1.0f, by - ay);
                            xa = fmaf((fmaxf(yb0, elo) - ay) * inv, bx - ax, ax);
                            xb = fmaf((fminf(yb1, ehi) - ay) * inv, bx - ax, ax);
                        }
                        xlo = fminf(xlo, fminf(xa, xb));
                        xhi = fmaxf(xhi, fmaxf(xa, xb));
                    }
                    if (xlo <= xhi) {
                        const int ix0 = max(0, fcell((xlo - g.eps) * g.inv_h, g.nx));
                        const int ix1 = min(g.nx - 1, fcell((xhi + g.eps) * g.inv_h, g.nx));
                        if (ix0 <= ix1) {
                            ixlo = ix0;
                            len = ix1 - ix0 + 1;
                        }
                    }
                }
                int incl = len;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int v = __shfl_up_sync(kFullG, incl, o);
                    if (lane >= o) incl += v;
                }
                const int total = __shfl_sync(kFullG, incl, 31);
                const int roff = ixlo - (incl - len);
                for (int cb = 0; cb < total; cb += 32) {
                    const int pos = cb + lane;
                    // row owning column position pos: first lane whose inclusive prefix exceeds it
                    int owner = 0;
#pragma unroll
                    for (int st = 16; st > 0; st >>= 1) {
                        const int v = __shfl_sync(kFullG, incl, owner + st - 1);
                        if (v <= pos) owner += st;
                    }
                    const int ix = pos + __shfl_sync(kFullG, roff, owner);
                    int b0 = 0, l0 = 0, b1 = 0, l1 = 0;
                    if (pos < total) {
                        const int cy = rbase + owner;
                        const float Zr = s_k[wid][0], f1r = s_k[wid][1], f2r = s_k[wid][2];
                        const float zrel = s_k[wid][5];
                        const float xc = fmaf((float)ix + 0.5f, g.h, -s_k[wid][3]);
                        const float yc = fmaf((float)cy + 0.5f, g.h, -s_k[wid][4]);
                        const float Zc = fmaf(f.c, xc, f.s * yc);
                        const float Xc = fmaf(f.ax, xc, f.bx * yc);
                        const float f1c = fmaf(g.kxh, Zc, -Xc), f2c = fmaf(g.kxh, Zc, Xc);
                        const float Zmin = Zc - Zr, Zmax = Zc + Zr;
                        const bool out = (Zmax < g.zn - g.eps) | (Zmin > g.zf + g.eps) | (f1c + f1r < -g.eps) |
                                         (f2c + f2r < -g.eps);
                        if (!out) {
                            const bool in_h = (Zmin >= g.zn + g.eps) & (Zmax <= g.zf - g.eps) &
                                              (f1c - f1r >= g.eps) & (f2c - f2r >= g.eps);
                            const float Zhi = fmaxf(fminf(Zmax, g.zf), 0.0f);
                            int c = fcell((zrel - g.kyd * Zhi - g.eps) * g.inv_hz, g.nz);
                            int dd = fcell((zrel + g.kyu * Zhi + g.eps) * g.inv_hz, g.nz) + 1;
                            c = min(max(c, 0), g.nz);
                            dd = min(max(dd, c), g.nz);
                            int a = c, b = c;
                            if (in_h) {
                                const float za = fminf(fmaxf((zrel - g.kyd * Zmin + g.eps) * g.inv_hz, -1.0f), g.nz + 1.0f);
                                const float zb = fminf(fmaxf((zrel + g.kyu * Zmin - g.eps) * g.inv_hz, -1.0f), g.nz + 1.0f);
                                a = min(max((int)ceilf(za), c), dd);
                                b = min(max((int)floorf(zb), a), dd);
                            }
                            // x-fastest tables: entry (cy, iz, ix) at (cy*(nz+1) + iz)*nx + ix
                            const int base = cy * (g.nz + 1) * g.nx + ix;
                            const int sc = gstart[base + c * g.nx], sa = gstart[base + a * g.nx];
                            const int sb = gstart[base + b * g.nx], sd = gstart[base + dd * g.nx];
                            if (b > a) {
                                const CellAgg hi = agg[base + b * g.nx], lo = agg[base + a * g.nx];
                                accq += hi.q - lo.q;
                                const long long hl = hi.hl - lo.hl;
                                acch += (int)(hl & 0xffffffffLL);
                                accl += (int)(hl >> 32);
                                if (kStats) nagg += (unsigned long long)(b - a);
                            }
                            b0 = sc; l0 = sa - sc;
                            b1 = sb; l1 = sd - sb;
                            if (kStats) {
                                ncol += 1;
                                if (!in_h) nstr += (unsigned long long)(l0 + l1);
                            }
                        }
                    }
                    // individual tests over this chunk's runs
                    if (kStats) ntest += (unsigned long long)(l0 + l1);
                    int pc = 0;
                    auto test = [&](int gi) {
                        const GRec G = grec[gi];
                        const long long q = guq[gi];
                        const bool v = visible_cs(f, cam, G.x, G.y, G.z, s_cs[wid], nref);
                        add_if(v, accq, q, pc, G.inc);
                        if (kStats) nvis += v;
                    };
                    // (1) long runs (straddling columns, mostly): one run at a time across the
                    //     whole warp, consecutive records per lane, no per-position search
                    {
                        const unsigned lm0 = __ballot_sync(kFullG, l0 >= kLongRun);
                        const unsigned lm1 = __ballot_sync(kFullG, l1 >= kLongRun);
#pragma unroll
                        for (int pass = 0; pass < 2; ++pass) {
                            unsigned lm = pass ? lm1 : lm0;
                            const int bb = pass ? b1 : b0, ll = pass ? l1 : l0;
                            while (lm) {
                                const int j = __ffs(lm) - 1;
                                lm &= lm - 1;
                                const int start = __shfl_sync(kFullG, bb, j);
                                const int len = __shfl_sync(kFullG, ll, j);
                                for (int o = lane; o < len; o += 32) test(start + o);
                            }
                        }
                        if (l0 >= kLongRun) l0 = 0;
                        if (l1 >= kLongRun) l1 = 0;
                    }
                    // (2) short runs packed into full windows: the owner lane of position gp is
                    //     the first lane whose inclusive prefix exceeds gp (warp binary search over
                    //     the prefixes held in registers), then its first or second run
                    const int sl = l0 + l1;
                    int ic = sl;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int v = __shfl_up_sync(kFullG, ic, o);
                        if (lane >= o) ic += v;
                    }
                    const int tot = __shfl_sync(kFullG, ic, 31);
                    const int ex = ic - sl;
                    for (int gb = 0; gb < tot; gb += 32) {
                        const int gp = gb + lane;
                        int lo = 0;
#pragma unroll
                        for (int st = 16; st > 0; st >>= 1) {
                            const int v = __shfl_sync(kFullG, ic, lo + st - 1);
                            if (v <= gp) lo += st;
                        }
                        const int eo = gp - __shfl_sync(kFullG, ex, lo);
                        const int lo0 = __shfl_sync(kFullG, l0, lo);
                        const int bo0 = __shfl_sync(kFullG, b0, lo);
                        const int bo1 = __shfl_sync(kFullG, b1, lo);
                        const int gi = eo < lo0 ? bo0 + eo : bo1 + (eo - lo0);
                        if (gp < tot) test(gi);
                    }
                    acch += pc & 0xffff;
                    accl += pc >> 16;
                    __syncwarp();
                }
            }
        }
        // warp totals (integers: exact, order-free)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            accq += __shfl_xor_sync(kFullG, accq, o);
            acch += __shfl_xor_sync(kFullG, acch, o);
            accl += __shfl_xor_sync(kFullG, accl, o);
        }
        if (lane == 0) {
            wp_gq[i] = accq;
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
            ncol += __shfl_xor_sync(kFullG, ncol, o);
            nstr += __shfl_xor_sync(kFullG, nstr, o);
            nvis += __shfl_xor_sync(kFullG, nvis, o);
        }
        if (lane == 0) {
            if (nref) atomicAdd(&stats[1], (unsigned long long)nref);
            atomicAdd(&stats[2], ntest);
            atomicAdd(&stats[3], nagg);
            atomicAdd(&stats[5], nstr);
            atomicAdd(&stats[6], ncol);
            atomicAdd(&stats[7], nvis);
        }
    }
}

int g_sms_g = 0, g_occ_g = 0;

}  // namespace

cudaError_t launch_gain_culled(rtg_map_s* m, rtg_traj_s* tr, const CamK& cam, const int* list, const int* count,
                               long long list_max, long long* wp_gq, int* wp_nh, int* wp_nl, int* counter,
                               unsigned long long* stats, cudaStream_t st) {
    if (!g_sms_g) {
        cudaDeviceGetAttribute(&g_sms_g, cudaDevAttrMultiProcessorCount, m->device);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_occ_g, k_gain_culled<false>, kWarpsG * 32, 0);
        if (g_occ_g < 1) g_occ_g = 1;
    }
    GainK g;
    g.ox = m->gg.ox; g.oy = m->gg.oy; g.oz = m->gg.oz; g.h = m->gg.hxy; g.hz = m->gg.hz; g.hh = 0.5f * m->gg.hxy;
    g.inv_h = 1.0f / m->gg.hxy; g.inv_hz = 1.0f / m->gg.hz;
    double ext = fmax(fmax(fabs(g.ox), fabs(g.oy)), fabs(g.oz)) +
                 (double)(m->gg.nx + m->gg.ny + m->gg.nz) * fmax(m->gg.hxy, m->gg.hz) + cam.zmid + cam.zhalf;
    g.eps = (float)(1e-3 + 256.0 * ldexp(1.0, -24) * ext);   // >> FP32 error of the cell tests
    g.nx = m->gg.nx; g.ny = m->gg.ny; g.nz = m->gg.nz;
    g.zn = cam.zmid - cam.zhalf; g.zf = cam.zmid + cam.zhalf;
    g.kxl = cam.kxh - cam.kxc; g.kxr = cam.kxh + cam.kxc;
    g.kyu = cam.kyh + cam.kyc; g.kyd = cam.kyh - cam.kyc;
    g.kxh = cam.kxh;
    long long blocks = (list_max + kWarpsG - 1) / kWarpsG;
    long long cap = (long long)g_sms_g * g_occ_g;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    if (stats)
        note_launch(), k_gain_culled<true><<<(unsigned)blocks, kWarpsG * 32, 0, st>>>(
            tr->x, tr->y, tr->z, tr->yaw, list, count, m->grec, m->guq, m->gstartT, m->gaggT, g, cam,
            wp_gq, wp_nh, wp_nl, counter, stats);
    else
        note_launch(), k_gain_culled<false><<<(unsigned)blocks, kWarpsG * 32, 0, st>>>(
            tr->x, tr->y, tr->z, tr->yaw, list, count, m->grec, m->guq, m->gstartT, m->gaggT, g, cam,
            wp_gq, wp_nh, wp_nl, counter, stats);
    return cudaGetLastError();
}

}  // namespace rtg
