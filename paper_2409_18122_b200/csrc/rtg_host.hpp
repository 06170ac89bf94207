// rtg_host.hpp -- host-side handle layouts and launch helpers of librtg (internal).
#pragma once
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>
#include <cuda_runtime.h>

#include "../../include/rtg.h"
#include "rtg_internal.cuh"

namespace rtg {

void set_error(const char* fmt, ...);

// launch accounting and optional CUDA-event profiling of the library's phases (rtg_api.cu)
void note_launch();
enum Phase { PH_MAP = 0, PH_CLASSIFY = 1, PH_COLLISION = 2, PH_LIST = 3, PH_GAIN = 4, PH_REDUCE = 5, PH_BEST = 6,
             PH_OTHER = 7 };
void prof_begin(int phase, cudaStream_t st);
void prof_end(int phase, cudaStream_t st);

// device-resident classification state (written by the classify kernels, read by the
// packing / reduction kernels; never read back on the scoring path)
struct ClassState {
    double tau_hi, tau_lo, mean, std;
    double scale;       // 2^S
    double inv_scale;   // 2^-S
    int shift;          // S
    int n_eligible;
};

struct GainGrid {
    float ox, oy, oz, hxy, hz;
    int nx, ny, nz;
    long long ncells;
};

struct ColGrid {
    float ox, oy, oz, h;
    int nx, ny, nz;
    long long ncells;
};


// scans (rtg_scan.cu): exclusive prefix of n values into out[0..n] (out[n] = total)
cudaError_t exclusive_scan_i32(const int* in, int* out, long long n, cudaStream_t st);
cudaError_t exclusive_scan_i64(const long long* in, long long* out, long long n, cudaStream_t st);
// device allocation through the stream-ordered pool
cudaError_t dev_alloc(void** p, size_t bytes, cudaStream_t st);
void dev_free(void* p, cudaStream_t st);
// (re)classification of a built map (rtg_map.cu)
rtg_status classify_map(rtg_map_s* m, int variant, double k_sigma, double tau_hi, double tau_lo,
                        cudaStream_t st);

}  // namespace rtg

struct rtg_map_s {
    int device = 0;
    cudaStream_t stream = nullptr;   // creation stream (release is enqueued on it)
    bool poisoned = false;
    long long n = 0, n_col = 0, n_gain = 0;
    rtg_robot robot{};
    // original-order inputs kept for (re)classification
    float* w_orig = nullptr;             // [n]
    unsigned char* flags = nullptr;      // [n] or null
    // visibility records (sorted by gain cell), padded to a multiple of kTile with NaN means
    long long n_gain_pad = 0;
    rtg::GRec* grec = nullptr;
    long long* guq = nullptr;            // fixed-point u per record
    int* gidx = nullptr;                 // original index per record
    int* gstart = nullptr;               // [ncells+1] first record of each gain cell, (iy, ix, iz) order
    // culled-kernel tables in x-fastest layout [iy][iz][ix], iz = 0..nz (iz = nz: column end), so
    // the lanes of a warp, which take neighbouring columns of a row, load neighbouring words
    long long ntab = 0;                  // ny * (nz + 1) * nx
    int* gstartT = nullptr;              // [ntab] first record of the cell (end of column at iz = nz)
    rtg::CellAgg* gaggT = nullptr;       // [ntab] exclusive prefixes (u_q, nH | nL << 32) there
    rtg::GainGrid gg{};
    // collision records (sorted by collision cell), padded likewise
    long long n_col_pad = 0;
    rtg::CRec* crec = nullptr;
    rtg::CMat* cmat = nullptr;
    rtg::CMat64* cmat64 = nullptr;
    int* cstart = nullptr;               // [ncells+1]
    rtg::ColGrid cg{};
    float rb_max = 0.f;
    float gq = 0.f;                      // FP32 collision guard
    // classification
    rtg::ClassState* cls = nullptr;      // device
    double* red_scratch = nullptr;       // device partials for the FP64 reductions
    int cls_variant = -1;
    double cls_k = 0, cls_th = 0, cls_tl = 0;
    bool cls_th_nan = true, cls_tl_nan = true;
    long long bytes = 0;
    std::vector<void*> allocs;
};

struct rtg_traj_s {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool poisoned = false;
    int K = 0, T = 0;
    float* x = nullptr;
    float* y = nullptr;
    float* z = nullptr;
    float* yaw = nullptr;
};
