// rtg_plan.cu -- planner bookkeeping on the device.
//
//  N4  uncertainty ledger: w_g = ||mu_k - mu_{k-1}||_2 for Gaussians whose mean
//      moved in the last map update, the previous value otherwise; the map's weights
//      are replaced in place and the map is reclassified without repacking its geometry.
//  N2  high-level guidance: region utility Omega = mean displacement per cuboidal
//      region (exact fixed-point sums, order free); viewpoints on the circle at the shortest
//      viewing distance around a region centroid, facing it; the
//      cost-benefit argmax of Omega / e^d.
// FP64 where a result is compared with the oracle's double arithmetic, with explicit
// round-to-nearest intrinsics so no contraction changes a rounding.
#include <climits>
#include <cmath>

#include "rtg_host.hpp"

namespace rtg {
namespace {

inline unsigned nblk(long long n, int t) {
    long long b = (n + t - 1) / t;
    return (unsigned)(b < 1 ? 1 : (b > 65535LL * 32 ? 65535LL * 32 : b));
}

// ---------------------------------------------------------------- N4 ledger
__global__ void k_ledger(long long n, const float* __restrict__ prev, const float* __restrict__ cur,
                         const float* __restrict__ wprev, float* __restrict__ wout) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const float a0 = prev[i], a1 = prev[n + i], a2 = prev[2 * n + i];
        const float b0 = cur[i], b1 = cur[n + i], b2 = cur[2 * n + i];
        if (a0 == b0 && a1 == b1 && a2 == b2) {
            wout[i] = wprev[i];
        } else {
            const double dx = __dsub_rn((double)b0, (double)a0), dy = __dsub_rn((double)b1, (double)a1);
            const double dz = __dsub_rn((double)b2, (double)a2);
            const double s = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
            wout[i] = __double2float_rn(__dsqrt_rn(s));
        }
    }
}

// validation of replacement weights (finite, >= 0): bad[0] |= 1
__global__ void k_check_w(long long n, const float* __restrict__ w, int* __restrict__ bad) {
    int b = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const float v = w[i];
        if (!(v >= 0.0f) || !isfinite(v)) b = 1;
    }
    if (__any_sync(0xffffffffu, b) && (threadIdx.x & 31) == 0) atomicOr(bad, 1);
}

// ---------------------------------------------------------------- N2 region utility
struct RegionK {
    double ox, oy, oz, size;
    int nx, ny, nz;
};

__device__ __forceinline__ int region_of(const GRec& r, const RegionK& g) {
    const int ix = (int)floor(__ddiv_rn(__dsub_rn((double)r.x, g.ox), g.size));
    const int iy = (int)floor(__ddiv_rn(__dsub_rn((double)r.y, g.oy), g.size));
    const int iz = (int)floor(__ddiv_rn(__dsub_rn((double)r.z, g.oz), g.size));
    if (ix < 0 || iy < 0 || iz < 0 || ix >= g.nx || iy >= g.ny || iz >= g.nz) return -1;
    return (iz * g.ny + iy) * g.nx + ix;
}

// pass 1: largest weight of a Gaussian inside the regions (non-negative floats order as ints)
// (also records each Gaussian's region for pass 2: the FP64 divisions run once)
__global__ void k_region_max(long long n, const GRec* __restrict__ rec, const int* __restrict__ gidx,
                             const float* __restrict__ w, RegionK g, int* __restrict__ wmax_bits, int* __restrict__ cnt,
                             int* __restrict__ rid) {
    int mx = 0, c = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int r = region_of(rec[i], g);
        rid[i] = r;
        if (r < 0) continue;
        mx = max(mx, __float_as_int(w[gidx[i]]));
        ++c;
    }
    mx = __reduce_max_sync(0xffffffffu, mx);
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0) {
        atomicMax(wmax_bits, mx);
        atomicAdd(cnt, c);
    }
}

// fixed-point scale 2^S with S = floor(52 - log2(M_total * w_max)): every region sum is an exact
// integer below 2^53 (in int64 here), so the sums do not depend on the accumulation order
__global__ void k_region_scale(const int* __restrict__ wmax_bits, const int* __restrict__ cnt, double* __restrict__ sc) {
    const double wm = (double)__int_as_float(*wmax_bits);
    const double tot = wm * (double)(*cnt);
    int s = 0;
    if (tot > 0.0) {
        s = (int)floor(52.0 - log2(tot));
        s = s > 1000 ? 1000 : (s < -1000 ? -1000 : s);
    }
    sc[0] = ldexp(1.0, s);
    sc[1] = ldexp(1.0, -s);
}

// pass 2: each thread walks kRegionRun consecutive records (copy B is sorted by visibility cell, so
// neighbours mostly share a region) and issues one pair of atomics per run of equal regions
constexpr int kRegionRun = 16;
__global__ void k_region_acc(long long n, const int* __restrict__ rid, const int* __restrict__ gidx,
                             const float* __restrict__ w, const double* __restrict__ sc,
                             unsigned long long* __restrict__ qsum, int* __restrict__ count) {
    const double scale = sc[0];
    const long long i0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * kRegionRun;
    if (i0 >= n) return;
    const long long i1 = min(n, i0 + kRegionRun);
    int cur = -1, c = 0;
    unsigned long long q = 0;
    for (long long i = i0; i < i1; ++i) {
        const int r = rid[i];
        if (r != cur) {
            if (cur >= 0) {
                atomicAdd(&qsum[cur], q);
                atomicAdd(&count[cur], c);
            }
            cur = r;
            q = 0;
            c = 0;
        }
        if (r >= 0) {
            q += (unsigned long long)llrint((double)w[gidx[i]] * scale);
            ++c;
        }
    }
    if (cur >= 0) {
        atomicAdd(&qsum[cur], q);
        atomicAdd(&count[cur], c);
    }
}

__global__ void k_region_final(long long nr, const unsigned long long* __restrict__ qsum, const int* __restrict__ count,
                               const double* __restrict__ sc, double* __restrict__ omega) {
    const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (r >= nr) return;
    const int c = count[r];
    omega[r] = c > 0 ? __ddiv_rn(__dmul_rn((double)qsum[r], sc[1]), (double)c) : 0.0;
}

// ---------------------------------------------------------------- N2 viewpoints
struct RingK {
    double d;      // viewing distance
    int R, n;
    float z;
};

__global__ void k_view_ring(RingK k, const float* __restrict__ cen, float* __restrict__ X, float* __restrict__ Y,
                            float* __restrict__ Z, float* __restrict__ Yaw) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= k.R * k.n) return;
    const int r = v / k.n, j = v - r * k.n;
    const double cx = cen[r], cy = cen[k.R + r];
    const double phi = __ddiv_rn(__dmul_rn(2.0 * M_PI, (double)j), (double)k.n);
    const double x = __dadd_rn(cx, __dmul_rn(k.d, cos(phi)));
    const double y = __dadd_rn(cy, __dmul_rn(k.d, sin(phi)));
    X[v] = __double2float_rn(x);
    Y[v] = __double2float_rn(y);
    Z[v] = k.z;
    Yaw[v] = __double2float_rn(atan2(__dsub_rn(cy, y), __dsub_rn(cx, x)));   // facing the centroid
}

// ---------------------------------------------------------------- N2 cost-benefit argmax
struct CbDev {
    double score;
    long long index;
};

__global__ void k_cost_benefit(const double* __restrict__ omega, const double* __restrict__ d, int K,
                               CbDev* __restrict__ out) {
    __shared__ double ss[1024], sd[1024];
    __shared__ int si[1024];
    double bs = -INFINITY, bd = INFINITY;
    int bi = -1;
    for (int j = threadIdx.x; j < K; j += blockDim.x) {   // j ascending per thread
        const double s = __ddiv_rn(omega[j], exp(d[j]));
        const double dj = d[j];
        if (bi < 0 || s > bs || (s == bs && dj < bd)) {
            bs = s;
            bd = dj;
            bi = j;
        }
    }
    ss[threadIdx.x] = bs;
    sd[threadIdx.x] = bd;
    si[threadIdx.x] = bi;
    __syncthreads();
    for (int h = blockDim.x / 2; h > 0; h >>= 1) {
        if ((int)threadIdx.x < h) {
            const int oi = si[threadIdx.x + h], mi = si[threadIdx.x];
            const double os = ss[threadIdx.x + h], ms = ss[threadIdx.x];
            const double od = sd[threadIdx.x + h], md = sd[threadIdx.x];
            const bool take = oi >= 0 && (mi < 0 || os > ms || (os == ms && (od < md || (od == md && oi < mi))));
            if (take) {
                ss[threadIdx.x] = os;
                sd[threadIdx.x] = od;
                si[threadIdx.x] = oi;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out->score = si[0] >= 0 ? ss[0] : -INFINITY;
        out->index = si[0];
    }
}

}  // namespace

// ---------------------------------------------------------------- launchers (rtg_api.cu)
cudaError_t launch_ledger(long long n, const float* prev, const float* cur, const float* wprev, float* wout,
                          cudaStream_t st) {
    if (n > 0) note_launch(), k_ledger<<<nblk(n, 256) > 4096 ? 4096 : nblk(n, 256), 256, 0, st>>>(n, prev, cur, wprev, wout);
    return cudaGetLastError();
}

cudaError_t launch_check_weights(long long n, const float* w, int* bad, cudaStream_t st) {
    if (n > 0) note_launch(), k_check_w<<<nblk(n, 256) > 4096 ? 4096 : nblk(n, 256), 256, 0, st>>>(n, w, bad);
    return cudaGetLastError();
}

cudaError_t launch_region_utility(rtg_map_s* m, const double origin[3], double size, const int dims[3], double* omega,
                                  int* count, cudaStream_t st) {
    RegionK g{origin[0], origin[1], origin[2], size, dims[0], dims[1], dims[2]};
    const long long nr = (long long)dims[0] * dims[1] * dims[2];
    char* scratch = nullptr;
    const size_t qb = sizeof(unsigned long long) * (size_t)nr;
    const long long ng = m->n_gain;
    cudaError_t e = dev_alloc((void**)&scratch, qb + 64 + sizeof(int) * (size_t)(ng > 0 ? ng : 1), st);
    if (e != cudaSuccess) return e;
    unsigned long long* qsum = (unsigned long long*)scratch;
    int* mx = (int*)(scratch + qb);
    int* cnt = mx + 1;
    double* sc = (double*)(scratch + qb + 16);
    int* rid = (int*)(scratch + qb + 64);
    e = cudaMemsetAsync(scratch, 0, qb + 64, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(count, 0, sizeof(int) * (size_t)nr, st);
    if (e != cudaSuccess) return e;
    const long long n = m->n_gain;   // copy B (gidx is parallel to it): the gain-eligible Gaussians
    const GRec* recB = m->grec + m->n_gain_pad;
    const unsigned nb = nblk(n, 256) > 2048 ? 2048 : nblk(n, 256);
    if (n > 0) {
        note_launch(), k_region_max<<<nb, 256, 0, st>>>(n, recB, m->gidx, m->w_orig, g, mx, cnt, rid);
        note_launch(), k_region_scale<<<1, 1, 0, st>>>(mx, cnt, sc);
        note_launch(), k_region_acc<<<nblk((n + kRegionRun - 1) / kRegionRun, 256), 256, 0, st>>>(
                           n, rid, m->gidx, m->w_orig, sc, qsum, count);
    } else {
        note_launch(), k_region_scale<<<1, 1, 0, st>>>(mx, cnt, sc);
    }
    note_launch(), k_region_final<<<nblk(nr, 256), 256, 0, st>>>(nr, qsum, count, sc, omega);
    e = cudaGetLastError();
    dev_free(scratch, st);
    return e;
}

cudaError_t launch_view_ring(int R, const float* cen, double d, int n, float z, rtg_traj_s* tr, cudaStream_t st) {
    RingK k{d, R, n, z};
    const int nv = R * n;
    note_launch(), k_view_ring<<<(nv + 255) / 256, 256, 0, st>>>(k, cen, tr->x, tr->y, tr->z, tr->yaw);
    return cudaGetLastError();
}

cudaError_t launch_cost_benefit(const double* omega, const double* d, int K, void* out_dev, cudaStream_t st) {
    note_launch(), k_cost_benefit<<<1, 1024, 0, st>>>(omega, d, K, (CbDev*)out_dev);
    return cudaGetLastError();
}

}  // namespace rtg
