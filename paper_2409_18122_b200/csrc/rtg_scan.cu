// rtg_scan.cu -- exclusive prefix sums used to build the cell grids (counting sort) and the
// exact fixed-point cell aggregates.  Three-phase block scan, recursive over block totals.
#include "rtg_host.hpp"

namespace rtg {
namespace {

constexpr int kScanThreads = 512;
constexpr int kScanPer = 8;
constexpr int kScanBlock = kScanThreads * kScanPer;   // elements per block

template <typename T>
__device__ T block_exclusive_scan(T v, T* sh, T& total) {
    // warp inclusive scan
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    T x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sh[wid] = x;
    __syncthreads();
    if (wid == 0) {
        T w = lane < (kScanThreads / 32) ? sh[lane] : T(0);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            T y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < (kScanThreads / 32)) sh[lane] = w;
    }
    __syncthreads();
    T warp_prefix = wid > 0 ? sh[wid - 1] : T(0);
    total = sh[kScanThreads / 32 - 1];
    __syncthreads();
    return warp_prefix + x - v;
}

// out[i] = sum_{j<i} in[j] within the block; block_sums[b] = block total
template <typename T>
__global__ void k_scan_local(const T* __restrict__ in, T* __restrict__ out, T* __restrict__ block_sums,
                             long long n) {
    __shared__ T sh[kScanThreads / 32];
    long long base = (long long)blockIdx.x * kScanBlock + (long long)threadIdx.x * kScanPer;
    T loc[kScanPer];
    T s = 0;
#pragma unroll
    for (int i = 0; i < kScanPer; ++i) {
        long long j = base + i;
        loc[i] = j < n ? in[j] : T(0);
        s += loc[i];
    }
    T total;
    T pre = block_exclusive_scan<T>(s, sh, total);
#pragma unroll
    for (int i = 0; i < kScanPer; ++i) {
        long long j = base + i;
        if (j < n) out[j] = pre;
        pre += loc[i];
    }
    if (threadIdx.x == 0 && block_sums) block_sums[blockIdx.x] = total;
}

template <typename T>
__global__ void k_scan_add(T* __restrict__ out, const T* __restrict__ offs, long long n) {
    long long base = (long long)blockIdx.x * kScanBlock + (long long)threadIdx.x * kScanPer;
    T o = offs[blockIdx.x];
#pragma unroll
    for (int i = 0; i < kScanPer; ++i) {
        long long j = base + i;
        if (j < n) out[j] += o;
    }
}

// out[n] = out[n-1] + in[n-1]
template <typename T>
__global__ void k_scan_tail(const T* __restrict__ in, T* __restrict__ out, long long n) {
    if (threadIdx.x == 0) out[n] = n > 0 ? out[n - 1] + in[n - 1] : T(0);
}

template <typename T>
cudaError_t scan_impl(const T* in, T* out, long long n, cudaStream_t st) {
    if (n <= 0) {
        note_launch(), k_scan_tail<T><<<1, 32, 0, st>>>(in, out, 0);
        return cudaGetLastError();
    }
    long long nb = (n + kScanBlock - 1) / kScanBlock;
    if (nb == 1) {
        note_launch(), k_scan_local<T><<<1, kScanThreads, 0, st>>>(in, out, nullptr, n);
    } else {
        T* sums = nullptr;
        cudaError_t e = dev_alloc((void**)&sums, sizeof(T) * (nb + 1), st);
        if (e != cudaSuccess) return e;
        note_launch(), k_scan_local<T><<<(unsigned)nb, kScanThreads, 0, st>>>(in, out, sums, n);
        // scan block totals in place (exclusive), recursively
        T* sums_scan = nullptr;
        e = dev_alloc((void**)&sums_scan, sizeof(T) * (nb + 1), st);
        if (e != cudaSuccess) return e;
        e = scan_impl<T>(sums, sums_scan, nb, st);
        if (e != cudaSuccess) return e;
        note_launch(), k_scan_add<T><<<(unsigned)nb, kScanThreads, 0, st>>>(out, sums_scan, n);
        dev_free(sums, st);
        dev_free(sums_scan, st);
    }
    note_launch(), k_scan_tail<T><<<1, 32, 0, st>>>(in, out, n);
    return cudaGetLastError();
}

}  // namespace

cudaError_t exclusive_scan_i32(const int* in, int* out, long long n, cudaStream_t st) {
    return scan_impl<int>(in, out, n, st);
}
cudaError_t exclusive_scan_i64(const long long* in, long long* out, long long n, cudaStream_t st) {
    return scan_impl<long long>(in, out, n, st);
}

}  // namespace rtg
