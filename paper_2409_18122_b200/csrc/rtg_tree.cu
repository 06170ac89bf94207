// rtg_tree.cu -- on-device motion-primitive tree (§IV-B2).
//
// Trajectory candidates are grown as a tree of unicycle motion primitives (fixed controls over dt,
// N_v x N_omega controls from [0, v_max] x [-omega_max, omega_max]), layer by layer:
// every frontier node is expanded by every control at once and ALL new collision samples of the
// layer are checked against the Gaussian map in one launch ("testing collisions of all sampled
// points with all Gaussians from the map at once while growing the search tree") -- one warp
// per primitive, the exact culled collision test of a4 per sample, stopping at the first collision.
// The search bookkeeping stays on the device too, so a whole plan is one stream of launches and one
// host synchronisation at the end:
//   - cost g = sum (lambda_t + v^2 + w^2) dt (Eq. low_level_planner with piecewise-constant u);
//   - a closed (x, y, heading) lattice keeping the lowest g (a device hash table).  Within a layer
//     the children are visited in creation order (node, then control): a child is kept iff its g is
//     below the lattice cell's value before the layer AND below every earlier child of the layer in
//     the same cell -- the children of a layer are grouped per cell through a per-layer hash table,
//     so this "strict prefix minimum" is exact whatever the thread order;
//   - goal region ||p - p_goal|| <= goal_radius: such nodes are candidates (not expanded);
//   - beam: the `beam` children of lowest f = g + h, h = ||p_goal - p|| / v_max, ties to
//     creation order -- an exact radix select in one CTA, then an ordered compaction;
//   - result: the n_traj cheapest candidates, or, when none reached the goal, the n_traj
//     nodes closest to it, ranked by (key, creation order), parents traced on device.
// Every double operation that decides a comparison is an explicit round-to-nearest intrinsic (no
// FMA contraction), so the decisions equal the FP64 oracle's (oracle/planning.py).
#include <algorithm>
#include <cmath>
#include <vector>

#include "rtg_host.hpp"

namespace rtg {
namespace {

constexpr unsigned long long kEmptyKey = ~0ull;
constexpr int kSelThreads = 1024;
constexpr int kMaxBeamWords = 4096;   // selection bits of up to 131,072 children per layer (k_beam)

// unicycle closed form from (x0, y0, th0) under (v, w) for time t, FP64 without
// contraction so the host oracle's rounding is reproduced
__device__ __forceinline__ void unicycle_at(double x0, double y0, double th0, double v, double w, double t,
                                            double& x, double& y, double& th) {
    th = __dadd_rn(th0, __dmul_rn(w, t));
    if (fabs(w) < 1e-12) {
        const double vt = __dmul_rn(v, t);
        x = __dadd_rn(x0, __dmul_rn(vt, cos(th0)));
        y = __dadd_rn(y0, __dmul_rn(vt, sin(th0)));
    } else {
        const double r = __ddiv_rn(v, w);
        x = __dadd_rn(x0, __dmul_rn(r, __dsub_rn(sin(th), sin(th0))));
        y = __dadd_rn(y0, __dmul_rn(r, __dsub_rn(cos(th0), cos(th))));
    }
}

__device__ __forceinline__ double wrap_pi(double a) {   // (-pi, pi]
    double r = remainder(a, 2.0 * M_PI);
    if (r <= -M_PI) r += 2.0 * M_PI;
    return r;
}

// search constants (host-computed once per plan)
struct TreeK {
    int P, S, beam, W;              // controls, samples per primitive, beam, beam * P
    double dt, gx, gy, r2, vmax;    // goal region and heuristic
    float z;
    int dedup;                      // lattice on
    double lxy, ldeg, rad2deg;      // lattice cell; 180 / pi
    long long amin, bmin, cmin;     // lattice index offsets
    int ba, bb;                     // bits of the packed b and c fields (a takes the rest)
    unsigned long long cmask;       // capacity - 1 of the closed table
    unsigned long long lmask;       // capacity - 1 of the per-layer table
};

// device state of one plan
struct Tree {
    double *nx, *ny, *nth, *ng;     // nodes (creation order), capacity NC
    double* nh;                     // their heuristic h (for the no-candidate ranking)
    int *npar, *ndep;
    int* frontier;                  // node ids, creation order, <= beam
    double *cx, *cy, *cth, *cg;     // children of the layer, index w = m * P + p
    unsigned char* cok;             // primitive collision-free
    unsigned long long* ckey;       // packed lattice key
    int *cslot, *cpos;              // per-layer cell slot and position in the slot's bucket
    int *acc, *rank, *cid;          // kept flag, its exclusive scan, node id
    unsigned long long* fkey;       // f bits of frontier-eligible children (else kEmptyKey)
    unsigned long long* tkey;       // closed lattice: key -> lowest g
    double* tval;
    unsigned long long* lkey;       // per-layer cells
    int *lcnt, *loff, *lbucket;
    int* cand;                      // candidate node ids (any order)
    int* cnt;                       // 0 M, 1 nodes, 2 candidates, 3 expanded, 4 error, 5 found, 6 reached
    int *sel, *order;               // final selection: node ids (any order), then ranked
    int *scanA, *scanB;             // per-layer scan scratch (cell counts, kept flags); NULL: allocate
    int zeroA, zeroB;               // their leading ints that k_expand clears
    unsigned long long *sa, *sb;    // their keys
    unsigned long long* fstat;      // this layer's eligible children: count, min key, max key (k_create)
};

__device__ __forceinline__ unsigned long long mix64(unsigned long long k) {   // splitmix64 finaliser
    k ^= k >> 30;
    k *= 0xbf58476d1ce4e5b9ull;
    k ^= k >> 27;
    k *= 0x94d049bb133111ebull;
    k ^= k >> 31;
    return k;
}

// lattice cell of a state (SPEC S:384 closed set): floor(x / lxy), floor(y / lxy),
// floor(th * 180/pi / ldeg), packed with host-derived offsets; error flag if out of range
__device__ __forceinline__ unsigned long long lattice_key(const TreeK& k, double x, double y, double th, int* err) {
    const long long a = (long long)floor(__ddiv_rn(x, k.lxy)) - k.amin;
    const long long b = (long long)floor(__ddiv_rn(y, k.lxy)) - k.bmin;
    const long long c = (long long)floor(__ddiv_rn(__dmul_rn(th, k.rad2deg), k.ldeg)) - k.cmin;
    if (a < 0 || b < 0 || c < 0 || b >= (1LL << k.ba) || c >= (1LL << k.bb) || a >= (1LL << (62 - k.ba - k.bb))) {
        atomicExch(err, 1);
        return 0;
    }
    return ((unsigned long long)a << (k.ba + k.bb)) | ((unsigned long long)b << k.bb) | (unsigned long long)c;
}

__device__ __forceinline__ double closed_get(const Tree& t, const TreeK& k, unsigned long long key) {
    for (unsigned long long s = mix64(key) & k.cmask;; s = (s + 1) & k.cmask) {
        const unsigned long long v = t.tkey[s];
        if (v == key) return t.tval[s];
        if (v == kEmptyKey) return INFINITY;
    }
}

__device__ __forceinline__ void closed_put(const Tree& t, const TreeK& k, unsigned long long key, double g) {
    for (unsigned long long s = mix64(key) & k.cmask;; s = (s + 1) & k.cmask) {
        const unsigned long long prev = atomicCAS(&t.tkey[s], kEmptyKey, key);
        if (prev == kEmptyKey || prev == key) {
            t.tval[s] = g;
            return;
        }
    }
}

__device__ __forceinline__ double h_of(const TreeK& k, double x, double y) {
    const double dx = __dsub_rn(k.gx, x), dy = __dsub_rn(k.gy, y);
    return __ddiv_rn(sqrt(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy))), k.vmax);
}

__device__ __forceinline__ bool at_goal(const TreeK& k, double x, double y) {
    const double dx = __dsub_rn(x, k.gx), dy = __dsub_rn(y, k.gy);
    return __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)) <= k.r2;
}

__device__ __forceinline__ unsigned long long dbits(double v) {   // order-preserving for v >= 0
    return (unsigned long long)__double_as_longlong(v);
}

// ---- root: node 0, its lattice cell, the first frontier (or the root is already a candidate)
__global__ void k_tree_init(Tree t, TreeK k, double x, double y, double th) {
    t.nx[0] = x; t.ny[0] = y; t.nth[0] = th; t.ng[0] = 0.0;
    t.nh[0] = h_of(k, x, y);
    t.npar[0] = -1; t.ndep[0] = 0;
    t.cnt[1] = 1;
    t.fstat[0] = 0; t.fstat[1] = kEmptyKey; t.fstat[2] = 0;
    if (k.dedup) closed_put(t, k, lattice_key(k, x, y, th, t.cnt + 4), 0.0);
    if (at_goal(k, x, y)) {
        t.cand[0] = 0;
        t.cnt[2] = 1;
        t.cnt[0] = 0;
    } else {
        t.frontier[0] = 0;
        t.cnt[0] = 1;
    }
}

// does any of the nj points held by lanes 0 .. nj-1 (px, py; height z) collide?  The candidates of
// the union of their cell boxes are loaded once and each is tested against every point: a Gaussian
// outside a point's own box lies beyond g.R > its bounding radius, so the sphere test rejects it for
// that point and every decision equals the one-point test (warp_point_collides).
__device__ bool warp_points_collide_any(float px, float py, float z, int nj, const CRec* __restrict__ crec,
                                        const CMat* __restrict__ cmat, const CSrc* __restrict__ csrc,
                                        const rtg_robot& rb, const int* __restrict__ cstart, const ColGridK& g,
                                        float gq, unsigned& nref, unsigned long long& ntest) {
    constexpr unsigned kAll = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const bool mine = lane < nj && isfinite(px) && isfinite(py) && isfinite(z);
    int ix0 = INT_MAX, ix1 = -1, iy0 = INT_MAX, iy1 = -1;
    if (mine) {
        ix0 = max(0, clamp_cell((px - g.R - g.ox) / g.h, 0, g.nx));
        ix1 = min(g.nx - 1, clamp_cell((px + g.R - g.ox) / g.h, 0, g.nx));
        iy0 = max(0, clamp_cell((py - g.R - g.oy) / g.h, 0, g.ny));
        iy1 = min(g.ny - 1, clamp_cell((py + g.R - g.oy) / g.h, 0, g.ny));
        if (ix0 > ix1 || iy0 > iy1) { ix0 = iy0 = INT_MAX; ix1 = iy1 = -1; }
    }
    const unsigned own = ix0 <= ix1 ? (unsigned)((ix1 - ix0 + 1) * (iy1 - iy0 + 1)) : 0u;
    const unsigned own_sum = __reduce_add_sync(kAll, own);
    ix0 = __reduce_min_sync(kAll, ix0);
    ix1 = __reduce_max_sync(kAll, ix1);
    iy0 = __reduce_min_sync(kAll, iy0);
    iy1 = __reduce_max_sync(kAll, iy1);
    const int iz0 = max(0, clamp_cell((z - g.R - g.oz) / g.h, 0, g.nz));
    const int iz1 = min(g.nz - 1, clamp_cell((z + g.R - g.oz) / g.h, 0, g.nz));
    if (ix0 > ix1 || iy0 > iy1 || iz0 > iz1) return false;
    const unsigned live = __ballot_sync(kAll, mine);
    // spread-out points (long primitives): the union box would hold many times the candidates of the
    // points' own boxes -- test them one at a time (same decisions, see warp_points_collide_mask)
    if ((long long)(ix1 - ix0 + 1) * (iy1 - iy0 + 1) > (long long)kUnionFactor * own_sum)
        return warp_points_collide_each(px, py, z, live, true, crec, cmat, csrc, rb, cstart, g, gq, nref, ntest) != 0u;
    const int nyr = iy1 - iy0 + 1;
    const int nrows = nyr * (iz1 - iz0 + 1);
    bool hit = false;
    for (int r0 = 0; r0 < nrows && !hit; r0 += 32) {
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
        for (int b0 = 0; b0 < total; b0 += 32) {
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
            bool h = false;
            for (unsigned lv = live; lv; lv &= lv - 1) {   // every live point (warp-uniform loop)
                const int jj = __ffs(lv) - 1;
                const float qx = __shfl_sync(kAll, px, jj), qy = __shfl_sync(kAll, py, jj);
                if (pos < total && !h) {
                    const float dx = qx - A.x, dy = qy - A.y, dz = z - A.z;
                    const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
                    if (d2 < A.rb2) h = collide_full(cmat[gi].m, dx, dy, dz, gq, &csrc[gi], rb, qx, qy, z, A.x, A.y, A.z, nref);
                }
            }
            ntest += (unsigned long long)min(32, total - b0) * __popc(live);
            if (__any_sync(kAll, h)) {
                hit = true;
                break;
            }
        }
        __syncwarp();
    }
    return hit;
}

// resident 256-thread blocks per SM for k_expand: 3 = 80 registers, spill-free (4 = 64 registers with
// spills measured 1 % slower at N = 5M, equal at 2M)
#ifndef RTG_EXPAND_MINB
#define RTG_EXPAND_MINB 3
#endif

// ---- expansion: one warp per (frontier node m, control p), all W = beam * P warps launched, those
// past M * P only clear their child.  Samples j = 1 .. S-1 at t_j = j dt / (S-1) (j = 0 is the
// parent's state, checked when it was created); ok = no sample collides; child = state at dt.
__global__ void __launch_bounds__(256, RTG_EXPAND_MINB) k_expand(Tree t, TreeK k, const double* __restrict__ ctl,
                                                const CRec* __restrict__ crec, const CMat* __restrict__ cmat,
                                                const CSrc* __restrict__ csrc, const rtg_robot rb,
                                                const int* __restrict__ cstart, ColGridK g, float gq, int n_col,
                                                unsigned long long* __restrict__ stats) {
    const int lane = threadIdx.x & 31;
    const long long gt = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (k.dedup && gt <= (long long)k.lmask) {   // this layer's cell table starts empty (W * 32 >= capacity)
        t.lkey[gt] = kEmptyKey;
        t.lcnt[gt] = 0;
    }
    if (t.scanA && gt < t.zeroA) t.scanA[gt] = 0;   // and so do this layer's scan tickets and flags
    if (t.scanB && gt < t.zeroB) t.scanB[gt] = 0;
    const long long w = gt >> 5;
    if (w >= k.W) return;
    const int M = t.cnt[0];
    if (w >= (long long)M * k.P) {
        if (lane == 0) t.cok[w] = 0;
        return;
    }
    const int m = (int)(w / k.P), p = (int)(w - (long long)m * k.P);
    const int par = t.frontier[m];
    const double x0 = t.nx[par], y0 = t.ny[par], th0 = t.nth[par];
    const double v = ctl[2 * p], om = ctl[2 * p + 1];
    unsigned nref = 0;
    unsigned long long ntest = 0;
    bool hit = false;
    int checked = 0;
    // the samples' states 32 at a time in parallel (lane l computes sample j0 + l: FP64 sin/cos once
    // per sample), then the warp tests them in order with the early exit; the last sample is the child
    double x = x0, y = y0, th = th0;
    for (int j0 = 1; j0 < k.S; j0 += 32) {
        double lx = x0, ly = y0, lth = th0;
        if (j0 + lane < k.S) {
            const double tt = __ddiv_rn(__dmul_rn((double)(j0 + lane), k.dt), (double)(k.S - 1));
            unicycle_at(x0, y0, th0, v, om, tt, lx, ly, lth);
        }
        const float sx = __double2float_rn(lx), sy = __double2float_rn(ly);
        const int nj = min(32, k.S - j0);
        if (!hit && n_col > 0) {   // the chunk's samples tested together (cok = no sample collides)
            hit = warp_points_collide_any(sx, sy, k.z, nj, crec, cmat, csrc, rb, cstart, g, gq, nref, ntest);
            checked += nj;
        }
        x = __shfl_sync(0xffffffffu, lx, nj - 1);
        y = __shfl_sync(0xffffffffu, ly, nj - 1);
        th = __shfl_sync(0xffffffffu, lth, nj - 1);
    }
    if (lane == 0) {
        t.cok[w] = hit ? 0 : 1;
        t.cx[w] = x;
        t.cy[w] = y;
        t.cth[w] = wrap_pi(th);
        t.cg[w] = __dadd_rn(t.ng[par], ctl[2 * k.P + p]);   // + the control's cost (after the controls)
        if (stats) {
            atomicAdd(&stats[0], (unsigned long long)checked);
            atomicAdd(&stats[1], ntest);
            if (nref) atomicAdd(&stats[2], (unsigned long long)nref);
        }
    }
}

// ---- lattice: each collision-free child joins its cell's bucket of this layer
__global__ void k_cells(Tree t, TreeK k) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= k.W || !t.cok[w]) return;
    const unsigned long long key = lattice_key(k, t.cx[w], t.cy[w], t.cth[w], t.cnt + 4);
    t.ckey[w] = key;
    for (unsigned long long s = mix64(key) & k.lmask;; s = (s + 1) & k.lmask) {
        const unsigned long long prev = atomicCAS(&t.lkey[s], kEmptyKey, key);
        if (prev == kEmptyKey || prev == key) {
            t.cslot[w] = (int)s;
            t.cpos[w] = atomicAdd(&t.lcnt[s], 1);
            return;
        }
    }
}

__global__ void k_bucket(Tree t, TreeK k) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= k.W || !t.cok[w]) return;
    t.lbucket[t.loff[t.cslot[w]] + t.cpos[w]] = w;
}

// kept iff g < min(closed value before the layer, g of every earlier child of the layer in the cell)
__global__ void k_keep(Tree t, TreeK k) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= k.W) return;
    int keep = t.cok[w];
    if (keep && k.dedup) {
        double lim = closed_get(t, k, t.ckey[w]);
        const int s = t.cslot[w], b0 = t.loff[s], n = t.lcnt[s];
        for (int i = 0; i < n; ++i) {
            const int o = t.lbucket[b0 + i];
            if (o < w) lim = fmin(lim, t.cg[o]);
        }
        keep = t.cg[w] < lim;
    }
    t.acc[w] = keep;
}

// the cell's last kept child (largest w; kept children have strictly decreasing g) writes its g
__global__ void k_close(Tree t, TreeK k) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= k.W || !t.acc[w]) return;
    const int s = t.cslot[w], b0 = t.loff[s], n = t.lcnt[s];
    for (int i = 0; i < n; ++i) {
        const int o = t.lbucket[b0 + i];
        if (o > w && t.acc[o]) return;
    }
    closed_put(t, k, t.ckey[w], t.cg[w]);
}

// kept children become nodes (ids in creation order); goal nodes are candidates, the others are
// eligible for the next frontier with key f = g + h
__global__ void k_create(Tree t, TreeK k, int depth) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long fk = kEmptyKey;
    if (w < k.W && t.acc[w]) {
        const int id = t.cnt[1] + t.rank[w];
        const double x = t.cx[w], y = t.cy[w], g = t.cg[w];
        t.nx[id] = x; t.ny[id] = y; t.nth[id] = t.cth[w]; t.ng[id] = g;
        t.npar[id] = t.frontier[w / k.P];
        t.ndep[id] = depth;
        t.cid[w] = id;
        const double h = h_of(k, x, y);
        t.nh[id] = h;
        if (at_goal(k, x, y)) t.cand[atomicAdd(&t.cnt[2], 1)] = id;
        else fk = dbits(__dadd_rn(g, h));
    }
    if (w < k.W) t.fkey[w] = fk;
    // the layer's eligible count and key range for k_beam (one atomic triple per warp)
    const bool el = fk != kEmptyKey && w < t.cnt[0] * k.P;
    const unsigned bal = __ballot_sync(0xffffffffu, el);
    if (bal == 0) return;
    unsigned long long lo = el ? fk : kEmptyKey, hi = el ? fk : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&t.fstat[0], (unsigned long long)__popc(bal));
        atomicMin(&t.fstat[1], lo);
        atomicMax(&t.fstat[2], hi);
    }
}

// ---- exact selection of the `need` smallest keys (a, b, id) among n items in one CTA: radix
// select, 11 bits per pass from the most significant digit of a, then b, then id (ids are unique,
// so it always ends exact).  Returns the decided prefix (pa, pb, pi under masks ma, mb, mi); an item
// is selected iff its masked key is below the prefix, or equal to it.
struct SelState {
    unsigned long long pa, pb, ma, mb;
    unsigned pi, mi;
};

constexpr int kRadixBits = 11, kRadixBins = 1 << kRadixBits;

// digit d of the concatenated key a(64) | b(64, optional) | id(32): the word, shift and width
__device__ __forceinline__ void digit_pos(int d, bool use_b, int& which, int& sh, int& wd) {
    const int na = 6, nb = use_b ? 6 : 0;   // 64 bits = 5 digits of 11 + one of 9
    int dd = d;
    int top = 64;
    which = 0;
    if (dd >= na) {
        dd -= na;
        which = 1;
        if (dd >= nb) {
            dd -= nb;
            which = 2;
            top = 32;
        }
    }
    const int hi = top - kRadixBits * dd;
    sh = hi > kRadixBits ? hi - kRadixBits : 0;
    wd = hi - sh;
}

template <typename Src>
__device__ SelState block_select(const Src& src, int n, int need, bool use_b) {
    __shared__ int hist[kRadixBins];
    __shared__ int s_wsum[kSelThreads / 32];
    __shared__ int s_need, s_done, s_t, s_before;
    __shared__ SelState s_st;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid == 0) {
        s_st = SelState{0, 0, 0, 0, 0, 0};
        s_need = need;
        s_done = 0;
    }
    __syncthreads();
    const int ndig = 6 + (use_b ? 6 : 0) + 3;
    for (int d = 0; d < ndig; ++d) {
        for (int j = tid; j < kRadixBins; j += blockDim.x) hist[j] = 0;
        __syncthreads();
        const SelState st = s_st;
        int which, sh, wd;
        digit_pos(d, use_b, which, sh, wd);
        const unsigned dmask = (1u << wd) - 1u;
        for (int i0 = tid; i0 < n; i0 += 4 * blockDim.x) {
            unsigned long long a[4], b[4];
            unsigned id[4];
            bool ok[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {   // four independent loads in flight
                const int i = i0 + u * blockDim.x;
                ok[u] = i < n && src.get(i, a[u], b[u], id[u]);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (!ok[u] || (a[u] & st.ma) != st.pa || (b[u] & st.mb) != st.pb || (id[u] & st.mi) != st.pi)
                    continue;
                const unsigned dg = which == 0 ? (unsigned)(a[u] >> sh) & dmask
                                               : (which == 1 ? (unsigned)(b[u] >> sh) & dmask : (id[u] >> sh) & dmask);
                atomicAdd(&hist[dg], 1);
            }
        }
        __syncthreads();
        // the bin where the running count reaches `need`: block scan, two bins per thread
        const int b0 = 2 * tid;
        const int h0 = hist[b0], h1 = hist[b0 + 1];
        int inc = h0 + h1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += u;
        }
        if (lane == 31) s_wsum[wid] = inc;
        __syncthreads();
        if (wid == 0) {
            const int v = s_wsum[lane];
            int w = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int u = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += u;
            }
            s_wsum[lane] = w - v;
        }
        __syncthreads();
        const int before = s_wsum[wid] + inc - (h0 + h1);   // items in bins < b0
        const int nd = s_need;
        if (before < nd && before + h0 >= nd) {
            s_t = b0;
            s_before = before;
        } else if (before + h0 < nd && before + h0 + h1 >= nd) {
            s_t = b0 + 1;
            s_before = before + h0;
        }
        __syncthreads();
        if (tid == 0) {
            const int t = s_t;
            s_need -= s_before;
            if (hist[t] == s_need) s_done = 1;
            SelState ns = s_st;
            const unsigned long long mk = (unsigned long long)dmask << sh;
            if (which == 0) {
                ns.pa |= (unsigned long long)t << sh;
                ns.ma |= mk;
            } else if (which == 1) {
                ns.pb |= (unsigned long long)t << sh;
                ns.mb |= mk;
            } else {
                ns.pi |= (unsigned)t << sh;
                ns.mi |= (unsigned)mk;
            }
            s_st = ns;
        }
        __syncthreads();
        if (s_done) break;
    }
    return s_st;
}

__device__ __forceinline__ bool selected(const SelState& s, unsigned long long a, unsigned long long b, unsigned id) {
    const unsigned long long xa = a & s.ma, xb = b & s.mb;
    if (xa != s.pa) return xa < s.pa;
    if (xb != s.pb) return xb < s.pb;
    return (id & s.mi) <= s.pi;
}

// exact selection of the `need` smallest (f, w) among the n children for the beam: the eligible keys
// all lie in [kmin, kmax], so their common bit prefix is decided before the first pass and the radix
// digits start at the highest bit where kmin and kmax differ; then the child index w (unique) decides
// ties.  Keys are read two per 16-byte load, eight loads in flight per thread; once at most kBeamCand
// items match the decided prefix, the pass that reads them also copies them to shared memory and the
// remaining passes read only that copy.
constexpr int kBeamCand = 1024;
__device__ SelState beam_select(const unsigned long long* __restrict__ fkey, int n, int need, int elig,
                                unsigned long long kmin, unsigned long long kmax) {
    __shared__ int hist[kRadixBins];
    __shared__ int s_wsum[kSelThreads / 32];
    __shared__ int s_need, s_done, s_t, s_before, s_match, s_nc, s_ncw;
    __shared__ SelState s_st;
    __shared__ unsigned long long s_ca[kBeamCand];
    __shared__ unsigned s_ci[kBeamCand];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    int top;   // bits still undecided: [top - 1 .. 0] of the 96-bit key f(64) | w(32)
    if (tid == 0) {
        SelState z{0, 0, 0, 0, 0, 0};
        const unsigned long long x = kmin ^ kmax;
        const int hb = x ? 64 - __clzll((long long)x) : 0;
        z.ma = hb == 64 ? 0ull : (~0ull << hb);
        z.pa = kmin & z.ma;
        s_st = z;
        s_need = need;
        s_done = 0;
        s_t = 32 + hb;
        s_match = elig;   // items matching the decided prefix
        s_nc = -1;        // shared-memory copy: not taken
        s_ncw = 0;
    }
    __syncthreads();
    top = s_t;
    const int npair = (n + 1) >> 1;
    const ulonglong2* f2 = reinterpret_cast<const ulonglong2*>(fkey);
    while (top > 0) {
        for (int j = tid; j < kRadixBins; j += blockDim.x) hist[j] = 0;
        __syncthreads();
        const SelState st = s_st;
        const int wd = top > 32 ? min(kRadixBits, top - 32) : min(kRadixBits, top);
        const int lo = top - wd;
        const unsigned dmask = (1u << wd) - 1u;
        const int nc = s_nc;
        const bool take = nc < 0 && s_match <= kBeamCand;
        for (int i = tid; i < nc; i += blockDim.x) {   // from the shared copy (nc < 0: skipped)
            const unsigned long long a = s_ca[i];
            const unsigned id = s_ci[i];
            if ((a & st.ma) != st.pa || (id & st.mi) != st.pi) continue;
            const unsigned dg = lo >= 32 ? (unsigned)(a >> (lo - 32)) & dmask : (id >> lo) & dmask;
            atomicAdd(&hist[dg], 1);
        }
        for (int j0 = tid; nc < 0 && j0 < npair; j0 += 8 * blockDim.x) {
            ulonglong2 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int j = j0 + u * blockDim.x;
                v[u] = j < npair ? f2[j] : make_ulonglong2(kEmptyKey, kEmptyKey);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const unsigned long long a = h ? v[u].y : v[u].x;
                    const unsigned id = (unsigned)(2 * (j0 + u * blockDim.x) + h);
                    if (a == kEmptyKey || (int)id >= n || (a & st.ma) != st.pa || (id & st.mi) != st.pi) continue;
                    const unsigned dg = lo >= 32 ? (unsigned)(a >> (lo - 32)) & dmask : (id >> lo) & dmask;
                    atomicAdd(&hist[dg], 1);
                    if (take) {
                        const int c = atomicAdd(&s_ncw, 1);
                        s_ca[c] = a;
                        s_ci[c] = id;
                    }
                }
            }
        }
        __syncthreads();
        const int b0 = 2 * tid;
        const int h0 = hist[b0], h1 = hist[b0 + 1];
        int inc = h0 + h1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += u;
        }
        if (lane == 31) s_wsum[wid] = inc;
        __syncthreads();
        if (wid == 0) {
            const int v = s_wsum[lane];
            int w = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int u = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += u;
            }
            s_wsum[lane] = w - v;
        }
        __syncthreads();
        const int before = s_wsum[wid] + inc - (h0 + h1);
        const int nd = s_need;
        if (before < nd && before + h0 >= nd) {
            s_t = b0;
            s_before = before;
        } else if (before + h0 < nd && before + h0 + h1 >= nd) {
            s_t = b0 + 1;
            s_before = before + h0;
        }
        __syncthreads();
        if (tid == 0) {
            const unsigned t = (unsigned)s_t;
            s_need -= s_before;
            if (hist[t] == s_need) s_done = 1;
            s_match = hist[t];
            if (take) s_nc = s_ncw;
            SelState ns = s_st;
            if (lo >= 32) {
                ns.pa |= (unsigned long long)t << (lo - 32);
                ns.ma |= (unsigned long long)dmask << (lo - 32);
            } else {
                ns.pi |= t << lo;
                ns.mi |= dmask << lo;
            }
            s_st = ns;
        }
        __syncthreads();
        if (s_done) break;
        top = lo;
    }
    return s_st;
}

// ---- next frontier (one CTA): layer totals, beam select, ordered compaction in creation order
__global__ void __launch_bounds__(kSelThreads) k_beam(Tree t, TreeK k) {
    __shared__ int s_warp[kSelThreads / 32];
    __shared__ int s_n;
    __shared__ unsigned long long s_fs[3];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid == 0) {
        const int M = t.cnt[0];
        s_n = M * k.P;                                  // this layer's children
        t.cnt[3] += M;
        t.cnt[1] += t.rank[k.W - 1] + t.acc[k.W - 1];   // nodes created by this layer
        // eligible count and key range gathered by k_create; cleared for the next layer
        s_fs[0] = t.fstat[0]; s_fs[1] = t.fstat[1]; s_fs[2] = t.fstat[2];
        t.fstat[0] = 0; t.fstat[1] = kEmptyKey; t.fstat[2] = 0;
    }
    __syncthreads();
    const int n = s_n;
    const bool all = s_fs[0] <= (unsigned long long)k.beam;
    SelState st{0, 0, 0, 0, 0, 0};
    if (!all) st = beam_select(t.fkey, n, k.beam, (int)s_fs[0], s_fs[1], s_fs[2]);
    // ordered compaction: warp w owns the contiguous children [c0, c1), 32 per ballot word; pass 1
    // keeps the selection bits in shared memory, pass 2 writes the selected node ids in order
    __shared__ unsigned s_bits[kMaxBeamWords];
    const bool use_bits = n <= 32 * kMaxBeamWords;
    const int nw = blockDim.x >> 5;
    const int per = ((n + nw - 1) / nw + 31) & ~31;
    const int c0 = min(n, wid * per), c1 = min(n, c0 + per);
    int cnt = 0;
    for (int b0 = c0; b0 < c1; b0 += 8 * 32) {
        unsigned long long f[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = b0 + 32 * u + lane;
            f[u] = i < c1 ? t.fkey[i] : kEmptyKey;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int b = b0 + 32 * u;
            const bool sel = f[u] != kEmptyKey && (all || selected(st, f[u], 0, (unsigned)(b + lane)));
            const unsigned bal = __ballot_sync(0xffffffffu, sel);
            if (b < c1) {
                if (lane == 0 && use_bits) s_bits[b >> 5] = bal;
                cnt += __popc(bal);
            }
        }
    }
    if (lane == 0) s_warp[wid] = cnt;
    __syncthreads();
    if (wid == 0) {
        const int v = lane < nw ? s_warp[lane] : 0;
        int w = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += u;
        }
        if (lane < nw) s_warp[lane] = w - v;
        if (lane == 31) t.cnt[0] = w;                  // the next frontier's size
    }
    __syncthreads();
    int pos = s_warp[wid];
    const unsigned lt = (1u << lane) - 1u;
    for (int b0 = c0; b0 < c1; b0 += 8 * 32) {   // eight words per step: their id loads in flight together
        unsigned bal[8];
        int id[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int b = b0 + 32 * u;
            if (b >= c1) {
                bal[u] = 0u;
            } else if (use_bits) {
                bal[u] = s_bits[b >> 5];
            } else {   // more children than the bit buffer holds: evaluate the selection again
                const int i = b + lane;
                const unsigned long long f = i < c1 ? t.fkey[i] : kEmptyKey;
                bal[u] = __ballot_sync(0xffffffffu, f != kEmptyKey && (all || selected(st, f, 0, (unsigned)i)));
            }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) id[u] = ((bal[u] >> lane) & 1u) ? t.cid[b0 + 32 * u + lane] : 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if ((bal[u] >> lane) & 1u) t.frontier[pos + __popc(bal[u] & lt)] = id[u];
            pos += __popc(bal[u]);
        }
    }
}

// ---- final selection (one CTA): the n_traj cheapest candidates by (g, id), or, with no candidate,
// the n_traj nodes (root excluded) closest to the goal by (h, g, id)
struct SrcCand {
    const int* cand;
    const double* ng;
    __device__ bool get(int i, unsigned long long& a, unsigned long long& b, unsigned& id) const {
        const int c = cand[i];
        a = dbits(ng[c]);
        b = 0;
        id = (unsigned)c;
        return true;
    }
};
struct SrcNodes {
    const double *nh, *ng;
    __device__ bool get(int i, unsigned long long& a, unsigned long long& b, unsigned& id) const {
        a = dbits(nh[i + 1]);
        b = dbits(ng[i + 1]);
        id = (unsigned)(i + 1);
        return true;
    }
};

template <typename Src>
__device__ void select_into(const Tree& t, const Src& src, int n, int need, bool use_b) {
    __shared__ int s_n;
    const bool all = n <= need;
    SelState st{0, 0, 0, 0, 0, 0};
    if (!all) st = block_select(src, n, need, use_b);
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        unsigned long long a, b;
        unsigned id;
        src.get(i, a, b, id);
        if (all || selected(st, a, b, id)) {
            const int j = atomicAdd(&s_n, 1);
            t.sel[j] = (int)id;
            t.sa[j] = a;
            t.sb[j] = b;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) t.cnt[5] = s_n;
}

__global__ void __launch_bounds__(kSelThreads) k_final(Tree t, TreeK k, int n_traj) {
    const int nc = t.cnt[2];
    if (threadIdx.x == 0) t.cnt[6] = nc > 0;
    if (nc > 0) select_into(t, SrcCand{t.cand, t.ng}, nc, n_traj, false);
    else select_into(t, SrcNodes{t.nh, t.ng}, t.cnt[1] - 1, n_traj, true);
}

// rank of each selected item by (a, b, id) -> order
__global__ void k_rank(Tree t) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int n = t.cnt[5];
    if (i >= n) return;
    const unsigned long long a = t.sa[i], b = t.sb[i];
    const int id = t.sel[i];
    int r = 0;
    for (int j = 0; j < n; ++j) {
        const unsigned long long aj = t.sa[j], bj = t.sb[j];
        r += aj < a || (aj == a && (bj < b || (bj == b && t.sel[j] < id)));
    }
    t.order[r] = id;
}

// waypoints of the ranked candidates: l = depth (l = 0: start; NaN past the candidate's last node)
__global__ void k_trace(Tree t, TreeK k, int T, float* wx, float* wy, float* wz, float* wyaw, double* cost) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= t.cnt[5]) return;
    int id = t.order[r];
    cost[r] = t.ng[id];
    for (; id >= 0; id = t.npar[id]) {
        const size_t l = (size_t)r * T + t.ndep[id];
        wx[l] = (float)t.nx[id];
        wy[l] = (float)t.ny[id];
        wz[l] = k.z;
        wyaw[l] = (float)t.nth[id];
    }
}

unsigned long long pow2_at_least(unsigned long long v) {
    unsigned long long p = 1;
    while (p < v) p <<= 1;
    return p;
}

int bits_for(long long range) {   // bits holding 0 .. range - 1
    int b = 0;
    while ((1LL << b) < range) ++b;
    return b;
}

}  // namespace

rtg_status plan_tree(rtg_map_s* m, const float start[3], const float goal[2], const rtg_tree_params& P,
                     cudaStream_t st, rtg_traj_s** out, double* cost, int* n_found, int* reached,
                     long long stats_out[4]) {
    // ---- controls: v on a uniform grid of [0, v_max] incl. endpoints, w likewise on
    // [-w_max, w_max]; a grid of one point is {v_max} / {0}.  Then the per-control costs.
    std::vector<double> ctl;
    for (int i = 0; i < P.n_v; ++i) {
        const double v = P.n_v == 1 ? (double)P.v_max : (double)P.v_max * (double)i / (double)(P.n_v - 1);
        for (int j = 0; j < P.n_omega; ++j) {
            const double w = P.n_omega == 1 ? 0.0
                                            : (double)P.omega_max * (double)(2 * j - (P.n_omega - 1)) /
                                                  (double)(P.n_omega - 1);
            ctl.push_back(v);
            ctl.push_back(w);
        }
    }
    const int NP = P.n_v * P.n_omega;
    for (int p = 0; p < NP; ++p)
        ctl.push_back(((double)P.lambda_t + ctl[2 * p] * ctl[2 * p] + ctl[2 * p + 1] * ctl[2 * p + 1]) * (double)P.dt);
    TreeK k{};
    k.P = NP;
    k.S = P.samples;
    k.beam = P.beam;
    k.W = P.beam * NP;
    k.dt = (double)P.dt;
    k.gx = goal[0];
    k.gy = goal[1];
    k.r2 = (double)P.goal_radius * (double)P.goal_radius;
    k.vmax = (double)P.v_max;
    k.z = P.z;
    k.dedup = P.lattice_xy > 0 && P.lattice_deg > 0;
    k.lxy = (double)P.lattice_xy;
    k.ldeg = (double)P.lattice_deg;
    k.rad2deg = 180.0 / M_PI;
    const long long NC = 1 + (long long)P.max_depth * k.W;
    if (NC >= (1LL << 31)) {
        set_error("rtg_plan_tree: 1 + max_depth * beam * controls must be < 2^31");
        return RTG_ERR_INVALID_ARGUMENT;
    }
    unsigned long long ccap = 2;
    const unsigned long long lcap = pow2_at_least(2ull * (unsigned long long)k.W);
    if (k.dedup) {
        // lattice indices reachable within max_depth primitives (arc length <= v_max dt each)
        const double reach = (double)P.max_depth * (double)P.v_max * (double)P.dt + 1.0;
        k.amin = (long long)std::floor(((double)start[0] - reach) / k.lxy) - 1;
        k.bmin = (long long)std::floor(((double)start[1] - reach) / k.lxy) - 1;
        k.cmin = (long long)std::floor(-180.0 / k.ldeg) - 1;
        const long long na = (long long)std::floor(((double)start[0] + reach) / k.lxy) + 2 - k.amin;
        const long long nb = (long long)std::floor(((double)start[1] + reach) / k.lxy) + 2 - k.bmin;
        const long long ncl = (long long)std::floor(180.0 / k.ldeg) + 2 - k.cmin;
        k.ba = bits_for(nb);
        k.bb = bits_for(ncl);
        if (bits_for(na) + k.ba + k.bb > 62) {
            set_error("rtg_plan_tree: lattice too fine for the reachable area (cell key exceeds 62 bits)");
            return RTG_ERR_INVALID_ARGUMENT;
        }
        const double cells = (double)na * (double)nb * (double)ncl;
        ccap = pow2_at_least((unsigned long long)std::min((double)NC, cells) * 2ull + 2ull);
    }
    k.cmask = ccap - 1;
    k.lmask = lcap - 1;
    // ---- device state (one allocation)
    const size_t W = (size_t)k.W, nc = (size_t)NC, nt = (size_t)P.n_traj, T = (size_t)P.max_depth + 1;
    size_t off = 0;
    auto carve = [&](size_t bytes) {
        const size_t o = off;
        off += (bytes + 255) & ~(size_t)255;
        return o;
    };
    const size_t o_n = carve(sizeof(double) * 5 * nc), o_pd = carve(sizeof(int) * 2 * nc);
    const size_t o_fr = carve(sizeof(int) * (size_t)k.beam), o_c = carve(sizeof(double) * 4 * W);
    const size_t o_ok = carve(W), o_key = carve(sizeof(unsigned long long) * W), o_i = carve(sizeof(int) * 5 * W);
    const size_t o_f = carve(sizeof(unsigned long long) * W);
    const size_t o_t = carve(sizeof(unsigned long long) * ccap), o_tv = carve(sizeof(double) * ccap);
    const size_t o_l = carve(sizeof(unsigned long long) * lcap), o_lc = carve(sizeof(int) * 2 * lcap);
    const size_t o_lb = carve(sizeof(int) * W), o_cand = carve(sizeof(int) * nc), o_cnt = carve(sizeof(int) * 8);
    const size_t o_sel = carve(sizeof(int) * 2 * nt), o_sab = carve(sizeof(unsigned long long) * 2 * nt);
    const size_t o_w = carve(sizeof(float) * 4 * nt * T), o_cost = carve(sizeof(double) * nt);
    const size_t o_ctl = carve(sizeof(double) * ctl.size()), o_st = carve(sizeof(unsigned long long) * 4);
    const size_t o_fs = carve(sizeof(unsigned long long) * 3);
    // the per-layer scans run from pre-cleared scratch when they fit one single-pass launch
    const bool fastA = (long long)lcap <= 64LL * 4096;
    const bool fastB = (long long)W <= 64LL * 4096;
    const size_t o_sa = carve(sizeof(int) * (size_t)scan_i32_scratch_ints((long long)lcap));
    const size_t o_sb = carve(sizeof(int) * (size_t)scan_i32_scratch_ints((long long)W));
    char* mem = nullptr;
    cudaError_t e = dev_alloc((void**)&mem, off, st);
    if (e != cudaSuccess) {
        set_error("rtg_plan_tree: %s", cudaGetErrorString(e));
        return e == cudaErrorMemoryAllocation ? RTG_ERR_OUT_OF_MEMORY : RTG_ERR_CUDA;
    }
    Tree t;
    t.nx = (double*)(mem + o_n); t.ny = t.nx + nc; t.nth = t.ny + nc; t.ng = t.nth + nc; t.nh = t.ng + nc;
    t.npar = (int*)(mem + o_pd); t.ndep = t.npar + nc;
    t.frontier = (int*)(mem + o_fr);
    t.cx = (double*)(mem + o_c); t.cy = t.cx + W; t.cth = t.cy + W; t.cg = t.cth + W;
    t.cok = (unsigned char*)(mem + o_ok);
    t.ckey = (unsigned long long*)(mem + o_key);
    t.cslot = (int*)(mem + o_i); t.cpos = t.cslot + W; t.acc = t.cpos + W; t.rank = t.acc + W; t.cid = t.rank + W;
    t.fkey = (unsigned long long*)(mem + o_f);
    t.tkey = (unsigned long long*)(mem + o_t); t.tval = (double*)(mem + o_tv);
    t.lkey = (unsigned long long*)(mem + o_l); t.lcnt = (int*)(mem + o_lc); t.loff = t.lcnt + lcap;
    t.lbucket = (int*)(mem + o_lb);
    t.cand = (int*)(mem + o_cand);
    t.cnt = (int*)(mem + o_cnt);
    t.sel = (int*)(mem + o_sel); t.order = t.sel + nt;
    t.sa = (unsigned long long*)(mem + o_sab); t.sb = t.sa + nt;
    t.fstat = (unsigned long long*)(mem + o_fs);
    t.scanA = fastA && k.dedup ? (int*)(mem + o_sa) : nullptr;
    t.scanB = fastB ? (int*)(mem + o_sb) : nullptr;
    t.zeroA = (int)scan_i32_zero_ints((long long)lcap);
    t.zeroB = (int)scan_i32_zero_ints((long long)W);
    float* wx = (float*)(mem + o_w);
    float *wy = wx + nt * T, *wz = wy + nt * T, *wyaw = wz + nt * T;
    double* d_cost = (double*)(mem + o_cost);
    double* d_ctl = (double*)(mem + o_ctl);
    unsigned long long* d_stats = (unsigned long long*)(mem + o_st);
    // ---- root (FP64 heading wrapped to (-pi, pi] like the oracle)
    double th0 = std::remainder((double)start[2], 2.0 * M_PI);
    if (th0 <= -M_PI) th0 += 2.0 * M_PI;
    e = cudaMemcpyAsync(d_ctl, ctl.data(), sizeof(double) * ctl.size(), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(d_stats, 0, sizeof(unsigned long long) * 4, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(t.cnt, 0, sizeof(int) * 8, st);
    if (e == cudaSuccess && k.dedup) e = cudaMemsetAsync(t.tkey, 0xff, sizeof(unsigned long long) * ccap, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(wx, 0xff, sizeof(float) * 4 * nt * T, st);   // all-ones: NaN
    if (e == cudaSuccess) note_launch(), k_tree_init<<<1, 1, 0, st>>>(t, k, (double)start[0], (double)start[1], th0),
        e = cudaGetLastError();
    ColGridK g;
    g.ox = m->cg.ox; g.oy = m->cg.oy; g.oz = m->cg.oz; g.h = m->cg.h;
    g.R = m->rb_max * (1.0f + 2e-5f) + 1e-4f;
    g.nx = m->cg.nx; g.ny = m->cg.ny; g.nz = m->cg.nz;
    const unsigned wblocks = (unsigned)((W * 32 + 255) / 256), tblocks = (unsigned)((W + 255) / 256);
    for (int depth = 1; depth <= P.max_depth && e == cudaSuccess; ++depth) {
        note_launch(), k_expand<<<wblocks, 256, 0, st>>>(t, k, d_ctl, m->crec, m->cmat, m->csrc, m->robot, m->cstart,
                                                          g, m->gq, (int)m->n_col, d_stats);
        e = cudaGetLastError();
        if (e == cudaSuccess && k.dedup) {
            note_launch(), k_cells<<<tblocks, 256, 0, st>>>(t, k), e = cudaGetLastError();
            if (e == cudaSuccess)
                e = t.scanA ? exclusive_scan_i32_into(t.lcnt, t.loff, (long long)lcap, t.scanA, st)
                            : exclusive_scan_i32(t.lcnt, t.loff, (long long)lcap, st);
            if (e == cudaSuccess) note_launch(), k_bucket<<<tblocks, 256, 0, st>>>(t, k), e = cudaGetLastError();
        }
        if (e == cudaSuccess) note_launch(), k_keep<<<tblocks, 256, 0, st>>>(t, k), e = cudaGetLastError();
        if (e == cudaSuccess && k.dedup) note_launch(), k_close<<<tblocks, 256, 0, st>>>(t, k), e = cudaGetLastError();
        if (e == cudaSuccess)
            e = t.scanB ? exclusive_scan_i32_into(t.acc, t.rank, (long long)W, t.scanB, st)
                        : exclusive_scan_i32(t.acc, t.rank, (long long)W, st);
        if (e == cudaSuccess) note_launch(), k_create<<<tblocks, 256, 0, st>>>(t, k, depth), e = cudaGetLastError();
        if (e == cudaSuccess) note_launch(), k_beam<<<1, kSelThreads, 0, st>>>(t, k), e = cudaGetLastError();
    }
    if (e == cudaSuccess) note_launch(), k_final<<<1, kSelThreads, 0, st>>>(t, k, P.n_traj), e = cudaGetLastError();
    const unsigned rblocks = (unsigned)((nt + 255) / 256);
    if (e == cudaSuccess) note_launch(), k_rank<<<rblocks, 256, 0, st>>>(t), e = cudaGetLastError();
    if (e == cudaSuccess)
        note_launch(), k_trace<<<rblocks, 256, 0, st>>>(t, k, (int)T, wx, wy, wz, wyaw, d_cost), e = cudaGetLastError();
    int hc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    unsigned long long hs[4] = {0, 0, 0, 0};
    std::vector<double> hcost(nt, 0.0);
    if (e == cudaSuccess) e = cudaMemcpyAsync(hc, t.cnt, sizeof(hc), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(hs, d_stats, sizeof(hs), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(hcost.data(), d_cost, sizeof(double) * nt, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    rtg_status s = RTG_OK;
    if (e != cudaSuccess) {
        set_error("rtg_plan_tree: %s", cudaGetErrorString(e));
        s = e == cudaErrorMemoryAllocation ? RTG_ERR_OUT_OF_MEMORY : RTG_ERR_CUDA;
    } else if (hc[4]) {
        set_error("rtg_plan_tree: lattice cell out of the reachable range");
        s = RTG_ERR_CUDA;
    } else {
        const int K = std::min(hc[5], P.n_traj);
        *n_found = K;
        *reached = hc[6];
        if (cost)
            for (int i = 0; i < K; ++i) cost[i] = hcost[i];
        if (stats_out) {
            stats_out[0] = hc[3];
            stats_out[1] = (long long)hc[1] - 1;
            stats_out[2] = (long long)hs[0];
            stats_out[3] = (long long)hs[1];
        }
        if (K == 0) {
            set_error("rtg_plan_tree: no collision-free primitive grows from the start");
            s = RTG_ERR_NO_FEASIBLE;
        } else {
            // the first K rows of the (k-major) scratch waypoints are the result
            s = rtg_traj_upload(m->device, K, (int)T, RTG_MEM_DEVICE, wx, wy, wz, wyaw, st, out);
        }
    }
    dev_free(mem, st);
    return s;
}

}  // namespace rtg
