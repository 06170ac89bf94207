// l2_peak.cu -- measured L2 -> SM read bandwidth of this B200 (the roof of k_gain_culled, whose
// records and tables are L2-resident: DRAM traffic is ~43 MB of ~58 GB read per launch).
//
// Three patterns over a buffer resident in L2 (warmed first, sizes well below the 126 MB L2):
//   seq    : every warp reads consecutive 512-byte blocks (LDG.128, one 16-byte item per lane);
//   seq_cg : the same with ld.global.cg (L1 bypass: L2 -> SM only);
//   runs   : the gain kernel's pattern -- 16-byte records in runs of R consecutive records that start
//            at random record offsets, 32 lanes take 32 consecutive items of the flattened runs.
// Timed with CUDA events over many passes; prints one JSON line.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_peak tools/l2_peak.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x)                                                                           \
    do {                                                                                \
        cudaError_t e_ = (x);                                                           \
        if (e_ != cudaSuccess) {                                                        \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            exit(1);                                                                    \
        }                                                                               \
    } while (0)

template <bool kCg>
__global__ void k_seq(const uint4* __restrict__ buf, long long n16, int passes, unsigned* __restrict__ sink) {
    const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long nth = (long long)gridDim.x * blockDim.x;
    unsigned acc = 0;
    for (int p = 0; p < passes; ++p) {
        // four independent loads in flight per thread (same addresses every pass: L2-resident)
        for (long long i = tid; i < n16; i += 4 * nth) {
            uint4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const long long j = i + u * nth;
                v[u] = make_uint4(0, 0, 0, 0);
                if (j < n16) {
                    if (kCg) {
                        asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                                     : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                                     : "l"(buf + j));
                    } else {
                        v[u] = __ldg(buf + j);
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
        }
    }
    if (acc == 0x9e3779b9u) sink[0] = acc;   // never true in practice: keeps the loads
}

// runs pattern: run r (of nruns) starts at record starts[r] and has R records; each warp walks a
// contiguous slice of the flattened item space, 32 items per step (one per lane), two steps per pass
template <int R>
__global__ void k_runs(const uint4* __restrict__ rec, const int* __restrict__ starts, int nitems, int passes,
                       unsigned* __restrict__ sink) {
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    unsigned acc = 0;
    for (int p = 0; p < passes; ++p) {
        for (int base = warp * 64; base < nitems; base += nwarps * 64) {
            const int ia = base + lane, ib = base + 32 + lane;
            const uint4 a = __ldg(rec + __ldg(starts + ia / R) + ia % R);
            const uint4 b = __ldg(rec + __ldg(starts + ib / R) + ib % R);
            acc ^= a.x ^ a.w ^ b.y ^ b.z;
        }
    }
    if (acc == 0x9e3779b9u) sink[0] = acc;
}


// ---- TMA variant of the runs pattern: per warp, each 64-item window's run segments are bulk-copied
// (cp.async.bulk, one per segment, issued by one lane each) into a shared-memory ring of NBUF windows
// tracked by one mbarrier per slot; the lanes then read items lane and lane + 32 of the window
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(unsigned long long* b, unsigned c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void bar_expect(unsigned long long* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(unsigned long long* b, unsigned parity) {
    asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra W_%=;\n\t}" ::"r"(su32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, unsigned bytes, unsigned long long* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(b)) : "memory");
}

template <int R, int NBUF, int WPB>
__global__ void __launch_bounds__(WPB * 32) k_runs_tma(const uint4* __restrict__ rec, const int* __restrict__ starts,
                                                       int nwin, int off, int passes, unsigned* __restrict__ sink) {
    __shared__ __align__(128) uint4 buf[WPB][NBUF][64];
    __shared__ __align__(8) unsigned long long bar[WPB][NBUF];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int warp = blockIdx.x * WPB + wid, nwarps = gridDim.x * WPB;
    if (lane < NBUF) bar_init(&bar[wid][lane], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    unsigned acc = 0;
    unsigned phase = 0;   // bit k: parity of slot k
    auto issue = [&](int w, int slot) {
        const int lo = w * 64 + off, hi = lo + 64;
        const int r0 = lo / R, r1 = (hi - 1) / R;
        if (lane == 0) bar_expect(&bar[wid][slot], 64 * 16);
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const int r = r0 + lane;
        if (r <= r1) {
            const int a = max(lo, r * R), b = min(hi, (r + 1) * R);
            bulk(&buf[wid][slot][a - lo], rec + __ldg(starts + r) + (a - r * R), (unsigned)(b - a) * 16u, &bar[wid][slot]);
        }
    };
    for (int p = 0; p < passes; ++p) {
        int k = 0;   // windows of this warp: w = warp + k * nwarps
        for (int j = 0; j < NBUF - 1 && warp + j * nwarps < nwin; ++j) issue(warp + j * nwarps, j);
        for (int w = warp; w < nwin; w += nwarps, ++k) {
            const int slot = k % NBUF;
            const int wn = w + (NBUF - 1) * nwarps;
            if (wn < nwin) issue(wn, (k + NBUF - 1) % NBUF);
            bar_wait(&bar[wid][slot], (phase >> slot) & 1u);
            phase ^= 1u << slot;
            const uint4 x = buf[wid][slot][lane], y = buf[wid][slot][lane + 32];
            acc ^= x.x ^ x.w ^ y.y ^ y.z;
            __syncwarp();
        }
    }
    if (acc == 0x9e3779b9u) sink[0] = acc;
}

int main(int argc, char** argv) {
    int dev = 0;
    CK(cudaSetDevice(dev));
    int sms = 0, clk_khz = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev));
    unsigned* sink;
    CK(cudaMalloc(&sink, 64));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    printf("{\"sms\": %d, \"results\": [", sms);
    bool first = true;
    const int threads = 256;
    // ---- sequential patterns over 8 .. 64 MB
    for (int cg = 0; cg < 2; ++cg) {
        for (long long mb : {8LL, 16LL, 32LL, 64LL}) {
            const long long bytes = mb << 20, n16 = bytes / 16;
            uint4* buf;
            CK(cudaMalloc(&buf, bytes));
            CK(cudaMemset(buf, 1, bytes));
            for (int bps : {4, 8}) {
                const int blocks = sms * bps;
                const int passes = (int)std::max(1LL, (40LL << 30) / bytes);   // ~40 GB per timing
                auto run = [&](int ps) {
                    if (cg) k_seq<true><<<blocks, threads>>>(buf, n16, ps, sink);
                    else k_seq<false><<<blocks, threads>>>(buf, n16, ps, sink);
                };
                run(2);
                CK(cudaDeviceSynchronize());
                float best = 1e30f;
                for (int rep = 0; rep < 3; ++rep) {
                    CK(cudaEventRecord(a));
                    run(passes);
                    CK(cudaEventRecord(b));
                    CK(cudaEventSynchronize(b));
                    float ms;
                    CK(cudaEventElapsedTime(&ms, a, b));
                    best = std::min(best, ms);
                }
                const double gbs = (double)bytes * passes / (best * 1e-3) / 1e9;
                printf("%s{\"pattern\": \"%s\", \"mb\": %lld, \"blocks_per_sm\": %d, \"GBps\": %.1f}", first ? "" : ", ",
                       cg ? "seq_cg" : "seq", mb, bps, gbs);
                first = false;
            }
            CK(cudaFree(buf));
        }
    }
    // ---- runs pattern: 2M 16-byte records (32 MB, the outdoor map's copy size), runs of R
    {
        const long long nrec = 2LL << 20;
        uint4* rec;
        CK(cudaMalloc(&rec, nrec * 16));
        CK(cudaMemset(rec, 3, nrec * 16));
        auto one = [&](int R, auto kern, int bps = 8, int thr = 256) {
            const long long nruns = (16LL << 20) / R;   // 16M items per pass (256 MB of records read)
            std::vector<int> hs(nruns);
            unsigned long long x = 88172645463325252ull;
            for (auto& s : hs) {
                x ^= x << 13; x ^= x >> 7; x ^= x << 17;
                s = (int)(x % (unsigned long long)(nrec - R));
            }
            int* ds;
            CK(cudaMalloc(&ds, nruns * sizeof(int)));
            CK(cudaMemcpy(ds, hs.data(), nruns * sizeof(int), cudaMemcpyHostToDevice));
            const int nitems = (int)(nruns * R);
            const int blocks = sms * bps;
            const int passes = 64;
            kern<<<blocks, thr>>>(rec, ds, nitems, 1, sink);
            CK(cudaDeviceSynchronize());
            float best = 1e30f;
            for (int rep = 0; rep < 3; ++rep) {
                CK(cudaEventRecord(a));
                kern<<<blocks, thr>>>(rec, ds, nitems, passes, sink);
                CK(cudaEventRecord(b));
                CK(cudaEventSynchronize(b));
                float ms;
                CK(cudaEventElapsedTime(&ms, a, b));
                best = std::min(best, ms);
            }
            // record bytes only (the start lookups, 4 bytes per R records, are not counted)
            const double gbs = (double)nitems * 16 * passes / (best * 1e-3) / 1e9;
            printf(", {\"pattern\": \"runs\", \"run_records\": %d, \"mb\": 32, \"warps_per_sm\": %d, \"GBps\": %.1f}", R,
                   bps * thr / 32, gbs);
            CK(cudaFree(ds));
        };
        auto tma = [&](int R, int nbuf, int wpb, int bps, auto kern) {
            const int off = 37;
            const long long nruns = (16LL << 20) / R;
            std::vector<int> hs(nruns);
            unsigned long long x = 88172645463325252ull;
            for (auto& s : hs) {
                x ^= x << 13; x ^= x >> 7; x ^= x << 17;
                s = (int)(x % (unsigned long long)(nrec - R));
            }
            int* ds;
            CK(cudaMalloc(&ds, nruns * sizeof(int)));
            CK(cudaMemcpy(ds, hs.data(), nruns * sizeof(int), cudaMemcpyHostToDevice));
            const int nwin = (int)((nruns * R - off) / 64);
            const int blocks = sms * bps;
            const int passes = 64;
            kern<<<blocks, wpb * 32>>>(rec, ds, nwin, off, 1, sink);
            CK(cudaDeviceSynchronize());
            float best = 1e30f;
            for (int rep = 0; rep < 3; ++rep) {
                CK(cudaEventRecord(a));
                kern<<<blocks, wpb * 32>>>(rec, ds, nwin, off, passes, sink);
                CK(cudaEventRecord(b));
                CK(cudaEventSynchronize(b));
                float ms;
                CK(cudaEventElapsedTime(&ms, a, b));
                best = std::min(best, ms);
            }
            const double gbs = (double)nwin * 64 * 16 * passes / (best * 1e-3) / 1e9;
            printf(", {\"pattern\": \"runs_tma\", \"run_records\": %d, \"nbuf\": %d, \"warps_per_sm\": %d, \"GBps\": %.1f}",
                   R, nbuf, wpb * bps, gbs);
            CK(cudaFree(ds));
        };
        tma(8, 2, 4, 9, k_runs_tma<8, 2, 4>);
        tma(8, 3, 4, 9, k_runs_tma<8, 3, 4>);
        tma(8, 4, 4, 9, k_runs_tma<8, 4, 4>);
        tma(16, 2, 4, 9, k_runs_tma<16, 2, 4>);
        tma(16, 3, 4, 9, k_runs_tma<16, 3, 4>);
        tma(16, 4, 4, 9, k_runs_tma<16, 4, 4>);
        tma(4, 3, 4, 9, k_runs_tma<4, 3, 4>);
        tma(64, 3, 4, 9, k_runs_tma<64, 3, 4>);
        tma(16, 3, 8, 8, k_runs_tma<16, 3, 8>);
        one(4, k_runs<4>);
        one(8, k_runs<8>);
        one(16, k_runs<16>);
        one(64, k_runs<64>);
        one(8, k_runs<8>, 9, 128);
        one(16, k_runs<16>, 9, 128);
        CK(cudaFree(rec));
    }
    printf("], \"clock_attr_mhz\": %.0f}\n", clk_khz / 1000.0);
    return 0;
}
