// rtg_scan.cu -- exclusive prefix sums used to build the cell grids (counting sort) and the
// exact fixed-point prefixes.  Single pass, decoupled look-back: tiles take ids in launch order
// from an atomic counter, publish their aggregate, then look back over their predecessors' published
// aggregates / inclusive prefixes (a warp examines 32 predecessors at a time) until an inclusive
// prefix closes the sum.  Integer sums are exact, so the result does not depend on the order.
#include "rtg_host.hpp"

namespace rtg {
namespace {

constexpr int kScanThreads = 512;
// elements per thread: 8 ints / 4 pairs, so the shared-memory stage (below) fits the static limit
template <typename T> struct ScanPer { static constexpr int v = sizeof(T) <= 4 ? 8 : 4; };
template <typename T> constexpr int scan_tile() { return kScanThreads * ScanPer<T>::v; }
// stage index with one pad word per 32: thread t's contiguous elements and the striped (coalesced)
// order both hit distinct banks
__device__ __forceinline__ int stage_ix(int q) { return q + (q >> 5); }

// a pair of 64-bit sums (u_q prefix, packed class counts) scanned together
struct I64x2 {
    long long a, b;
    I64x2() = default;
    __host__ __device__ I64x2(long long x) : a(x), b(x) {}
    __host__ __device__ I64x2(long long x, long long y) : a(x), b(y) {}
    __host__ __device__ I64x2& operator+=(const I64x2& o) { a += o.a; b += o.b; return *this; }
    __host__ __device__ I64x2 operator+(const I64x2& o) const { return I64x2(a + o.a, b + o.b); }
    __host__ __device__ I64x2 operator-(const I64x2& o) const { return I64x2(a - o.a, b - o.b); }
};
__device__ __forceinline__ int shfl_up(int v, int o) { return __shfl_up_sync(0xffffffffu, v, o); }
__device__ __forceinline__ I64x2 shfl_up(I64x2 v, int o) {
    return I64x2(__shfl_up_sync(0xffffffffu, v.a, o), __shfl_up_sync(0xffffffffu, v.b, o));
}
__device__ __forceinline__ int shfl_down(int v, int o) { return __shfl_down_sync(0xffffffffu, v, o); }
__device__ __forceinline__ I64x2 shfl_down(I64x2 v, int o) {
    return I64x2(__shfl_down_sync(0xffffffffu, v.a, o), __shfl_down_sync(0xffffffffu, v.b, o));
}

// L2 loads of other tiles' published values (never a stale L1 line)
__device__ __forceinline__ int load_cg(const int* p) { return __ldcg(p); }
__device__ __forceinline__ I64x2 load_cg(const I64x2* p) {
    const long long* q = reinterpret_cast<const long long*>(p);
    return I64x2(__ldcg(q), __ldcg(q + 1));
}

template <typename T>
__device__ T block_exclusive_scan(T v, T* sh, T& total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    T x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = shfl_up(x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sh[wid] = x;
    __syncthreads();
    if (wid == 0) {
        T w = lane < (kScanThreads / 32) ? sh[lane] : T(0);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            T y = shfl_up(w, o);
            if (lane >= o) w += y;
        }
        if (lane < (kScanThreads / 32)) sh[lane] = w;
    }
    __syncthreads();
    T warp_prefix = wid > 0 ? sh[wid - 1] : T(0);
    total = sh[kScanThreads / 32 - 1];
    return warp_prefix + x - v;
}

// status of tile t: flag[t] = 0 (nothing yet), 1 (aggregate published), 2 (inclusive prefix
// published); the value is written before the flag, separated by a fence
// input loaders
template <typename T>
struct LoadArr {
    const T* __restrict__ p;
    __device__ T operator()(long long j) const { return p[j]; }
};
// column (iy, x) of the visibility grid -> its records over all z-cells, from the z-fastest table
// [ny][nx + 1][nz] whose entries start with the first record of cell (iy, iz, x) (x + 1: its end);
// `stride` ints per entry
struct LoadColCount {
    const int* __restrict__ tab;
    int nx, nz, stride;
    __device__ int operator()(long long col) const {
        const long long iy = col / nx, x = col - iy * nx;
        const int* t = tab + (iy * (nx + 1) + x) * nz * stride;
        int c = 0;
        for (int iz = 0; iz < nz; ++iz) c += t[(nz + iz) * stride] - t[iz * stride];
        return c;
    }
};
// copy-B record -> (u_q, packed class count nH | nL << 32)
struct LoadUc {
    const GRec* __restrict__ p;
    __device__ I64x2 operator()(long long j) const {
        const unsigned uc = p[j].uc;
        const unsigned c = uc >> kUqBits;
        return I64x2((long long)(uc & kUqMask), c == kClsH ? 1LL : (c == kClsL ? (1LL << 32) : 0LL));
    }
};

template <typename T, typename Load>
__global__ void __launch_bounds__(kScanThreads) k_scan(Load in, T* __restrict__ out, long long n,
                                                        int* __restrict__ ticket, volatile int* flag, T* agg, T* inc) {
    constexpr int PER = ScanPer<T>::v, TILE = scan_tile<T>();
    __shared__ T sh[kScanThreads / 32];
    __shared__ T s_prefix;
    __shared__ int s_tile;
    __shared__ T stage[TILE + TILE / 32];
    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1);
    __syncthreads();
    const int tile = s_tile;
    const long long tbase = (long long)tile * TILE;
    // coalesced load of the tile into shared memory, then each thread takes PER consecutive elements
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int q = i * kScanThreads + threadIdx.x;
        const long long j = tbase + q;
        stage[stage_ix(q)] = j < n ? in(j) : T(0);
    }
    __syncthreads();
    T loc[PER];
    T s = T(0);
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        loc[i] = stage[stage_ix(threadIdx.x * PER + i)];
        s += loc[i];
    }
    T total;
    T pre = block_exclusive_scan<T>(s, sh, total);
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        if (tile == 0) {
            if (lane == 0) {
                inc[0] = total;
                __threadfence();
                flag[0] = 2;
                s_prefix = T(0);
            }
        } else {
            if (lane == 0) {
                agg[tile] = total;
                __threadfence();
                flag[tile] = 1;
            }
            // look back over predecessors tile-1-lane, 32 at a time
            T run = T(0);
            int look = tile - 1;
            for (;;) {
                const int p = look - lane;
                int f = 2;
                if (p >= 0) {
                    do { f = flag[p]; } while (f == 0);
                }
                __threadfence();
                const unsigned closed = __ballot_sync(0xffffffffu, f == 2);   // lanes at an inclusive prefix
                const int stop = closed ? __ffs(closed) - 1 : 31;           // nearest one (p >= 0 has one by tile 0)
                T v = T(0);
                if (p >= 0 && lane <= stop) v = (f == 2) ? load_cg(inc + p) : load_cg(agg + p);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += shfl_down(v, o);
                run += v;   // lane 0 holds the warp sum
                if (closed) break;
                look -= 32;
            }
            if (lane == 0) {
                inc[tile] = run + total;
                __threadfence();
                flag[tile] = 2;
                s_prefix = run;
            }
        }
    }
    __syncthreads();
    pre += s_prefix;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        stage[stage_ix(threadIdx.x * PER + i)] = pre;
        pre += loc[i];
        if (tbase + threadIdx.x * PER + i == n - 1) out[n] = pre;   // total
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < PER; ++i) {   // coalesced store
        const int q = i * kScanThreads + threadIdx.x;
        const long long j = tbase + q;
        if (j < n) out[j] = stage[stage_ix(q)];
    }
}

template <typename T>
__global__ void k_scan_empty(T* out) { out[0] = T(0); }

// ---- large inputs: reduce-then-scan (no serial look-back chain over thousands of tiles)
// pass 1: per-tile sums (coalesced, striped)
template <typename T, typename Load>
__global__ void __launch_bounds__(kScanThreads) k_tile_sums(Load in, long long n, T* __restrict__ sums) {
    constexpr int PER = ScanPer<T>::v, TILE = scan_tile<T>();
    __shared__ T sh[kScanThreads / 32];
    const long long tbase = (long long)blockIdx.x * TILE;
    T s = T(0);
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const long long j = tbase + i * kScanThreads + threadIdx.x;
        if (j < n) s += in(j);
    }
    T total;
    block_exclusive_scan<T>(s, sh, total);
    if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

// pass 2: exclusive scan of the tile sums in one block (sums[nt] = grand total)
template <typename T>
__global__ void __launch_bounds__(kScanThreads) k_scan_sums(T* __restrict__ sums, int nt) {
    __shared__ T sh[kScanThreads / 32];
    __shared__ T s_carry;
    if (threadIdx.x == 0) s_carry = T(0);
    __syncthreads();
    for (int b = 0; b < nt; b += kScanThreads) {
        const int i = b + threadIdx.x;
        const T v = i < nt ? sums[i] : T(0);
        T total;
        const T ex = block_exclusive_scan<T>(v, sh, total);
        const T carry = s_carry;
        if (i < nt) sums[i] = carry + ex;
        __syncthreads();
        if (threadIdx.x == 0) s_carry = carry + total;
        __syncthreads();
    }
    if (threadIdx.x == 0) sums[nt] = s_carry;
}

// pass 3: each tile rescans its elements (staged, coalesced) from its offset
template <typename T, typename Load>
__global__ void __launch_bounds__(kScanThreads) k_tile_apply(Load in, T* __restrict__ out, long long n,
                                                             const T* __restrict__ sums, int nt) {
    constexpr int PER = ScanPer<T>::v, TILE = scan_tile<T>();
    __shared__ T sh[kScanThreads / 32];
    __shared__ T stage[TILE + TILE / 32];
    const long long tbase = (long long)blockIdx.x * TILE;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int q = i * kScanThreads + threadIdx.x;
        const long long j = tbase + q;
        stage[stage_ix(q)] = j < n ? in(j) : T(0);
    }
    __syncthreads();
    T loc[PER];
    T s = T(0);
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        loc[i] = stage[stage_ix(threadIdx.x * PER + i)];
        s += loc[i];
    }
    T total;
    T pre = block_exclusive_scan<T>(s, sh, total) + sums[blockIdx.x];
    __syncthreads();
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        stage[stage_ix(threadIdx.x * PER + i)] = pre;
        pre += loc[i];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int q = i * kScanThreads + threadIdx.x;
        const long long j = tbase + q;
        if (j < n) out[j] = stage[stage_ix(q)];
    }
    if (blockIdx.x == nt - 1 && threadIdx.x == 0) out[n] = sums[nt];   // total
}

// up to this many tiles the single-pass look-back scan (one launch); beyond, reduce-then-scan (the
// look-back chain over thousands of concurrently running tiles costs more than two extra launches)
constexpr long long kChainTiles = 64;

template <typename T, typename Load>
cudaError_t scan_impl(Load in, T* out, long long n, cudaStream_t st) {
    if (n <= 0) {
        note_launch(), k_scan_empty<T><<<1, 1, 0, st>>>(out);
        return cudaGetLastError();
    }
    const long long nt = (n + scan_tile<T>() - 1) / scan_tile<T>();
    if (nt >= (1LL << 31)) return cudaErrorInvalidValue;
    if (nt > kChainTiles) {
        T* sums = nullptr;
        cudaError_t e = dev_alloc((void**)&sums, sizeof(T) * (size_t)(nt + 1), st);
        if (e != cudaSuccess) return e;
        note_launch(), k_tile_sums<T, Load><<<(unsigned)nt, kScanThreads, 0, st>>>(in, n, sums);
        note_launch(), k_scan_sums<T><<<1, kScanThreads, 0, st>>>(sums, (int)nt);
        note_launch(), k_tile_apply<T, Load><<<(unsigned)nt, kScanThreads, 0, st>>>(in, out, n, sums, (int)nt);
        e = cudaGetLastError();
        dev_free(sums, st);
        return e;
    }
    // scratch: ticket + flags (zeroed), aggregates, inclusive prefixes
    const size_t fb = sizeof(int) * (size_t)(nt + 1), vb = sizeof(T) * (size_t)nt;
    char* mem = nullptr;
    cudaError_t e = dev_alloc((void**)&mem, ((fb + 255) & ~(size_t)255) + 2 * vb + 64, st);
    if (e != cudaSuccess) return e;
    int* ticket = (int*)mem;
    int* flags = ticket + 1;
    T* agg = (T*)(mem + ((fb + 255) & ~(size_t)255));
    T* inc = agg + nt;
    e = cudaMemsetAsync(mem, 0, fb, st);
    if (e != cudaSuccess) return e;
    note_launch(), k_scan<T, Load><<<(unsigned)nt, kScanThreads, 0, st>>>(in, out, n, ticket, flags, agg, inc);
    e = cudaGetLastError();
    dev_free(mem, st);
    return e;
}

}  // namespace

cudaError_t exclusive_scan_i32(const int* in, int* out, long long n, cudaStream_t st) {
    return scan_impl<int>(LoadArr<int>{in}, out, n, st);
}

// single-pass scan into caller scratch (scan_i32_scratch_ints(n) ints, of which the first
// scan_i32_zero_ints(n) must be zero at launch): one launch, no allocation -- for the per-layer scans
// of rtg_plan_tree, whose scratch is cleared by the preceding kernel.  n <= kChainTiles tiles.
long long scan_i32_tiles(long long n) { return (n + scan_tile<int>() - 1) / scan_tile<int>(); }
long long scan_i32_zero_ints(long long n) { return scan_i32_tiles(n) + 1; }
long long scan_i32_scratch_ints(long long n) { return scan_i32_zero_ints(n) + 2 * scan_i32_tiles(n); }
cudaError_t exclusive_scan_i32_into(const int* in, int* out, long long n, int* scratch, cudaStream_t st) {
    const long long nt = scan_i32_tiles(n);
    if (n <= 0 || nt > kChainTiles) return cudaErrorInvalidValue;
    int* ticket = scratch;
    int* flags = ticket + 1;
    int* agg = flags + nt;
    int* inc = agg + nt;
    note_launch(), k_scan<int, LoadArr<int>><<<(unsigned)nt, kScanThreads, 0, st>>>(LoadArr<int>{in}, out, n, ticket,
                                                                                   flags, agg, inc);
    return cudaGetLastError();
}
cudaError_t exclusive_scan_col_counts(const int* tab, int stride, int nx, int nz, long long ncols, int* out,
                                      cudaStream_t st) {
    return scan_impl<int>(LoadColCount{tab, nx, nz, stride}, out, ncols, st);
}
cudaError_t exclusive_scan_i64x2(const long long* in, long long* out, long long n, cudaStream_t st) {
    return scan_impl<I64x2>(LoadArr<I64x2>{reinterpret_cast<const I64x2*>(in)}, reinterpret_cast<I64x2*>(out), n, st);
}
cudaError_t exclusive_scan_grec_uc(const GRec* rec, long long* out, long long n, cudaStream_t st) {
    return scan_impl<I64x2>(LoadUc{rec}, reinterpret_cast<I64x2*>(out), n, st);
}

}  // namespace rtg
