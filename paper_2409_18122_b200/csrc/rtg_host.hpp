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

// visibility grid: rows (hy) x x-cells (hx) x z-cells (hz) over the bounding box of the
// gain-eligible means.  Two record copies are sorted by it: copy A by (iy, ix) (whole columns,
// used for the horizontally straddling flanks of a row), copy B by (iy, iz, ix) (a row's z-slab
// is x-contiguous, used for the horizontally inside part of a row, z-cell by z-cell).
struct GainGrid {
    float ox, oy, oz, hx, hy, hz;
    int nx, ny, nz;
    int nxb;             // x-blocks of kZoccX cells (z-occupancy table)
    long long ncellsA;   // ny * nx
    long long ncellsB;   // ny * nz * nx
};

struct ColGrid {
    float ox, oy, oz, h;
    int nx, ny, nz;
    long long ncells;
};


// scans (rtg_scan.cu): exclusive prefix of n values into out[0..n] (out[n] = total)
cudaError_t exclusive_scan_i32(const int* in, int* out, long long n, cudaStream_t st);
// single-pass scan into caller scratch whose first scan_i32_zero_ints(n) ints are zero (n small)
long long scan_i32_zero_ints(long long n);
long long scan_i32_scratch_ints(long long n);
cudaError_t exclusive_scan_i32_into(const int* in, int* out, long long n, int* scratch, cudaStream_t st);
// pairs of 64-bit sums (in: 2n long longs; out: 2(n + 1), the total last)
cudaError_t exclusive_scan_i64x2(const long long* in, long long* out, long long n, cudaStream_t st);
// copy-B records' (u_q, nH | nL << 32) pairs (from GRec::uc) scanned into out[0 .. 2n+1]
cudaError_t exclusive_scan_grec_uc(const GRec* rec, long long* out, long long n, cudaStream_t st);
// exclusive scan over the ncols = ny * nx columns (row-major) of their record counts (all z-cells), read
// from the z-fastest table [ny][nx + 1][nz] of `stride`-int entries led by the cell's first record;
// out[ncols] = total
cudaError_t exclusive_scan_col_counts(const int* tab, int stride, int nx, int nz, long long ncols, int* out,
                                      cudaStream_t st);
// device allocation through the stream-ordered pool
cudaError_t dev_alloc(void** p, size_t bytes, cudaStream_t st);
void dev_free(void* p, cudaStream_t st);
// frees a stream-ordered device block on every return path (the early error returns included)
struct DevFreeGuard {
    void** p;
    cudaStream_t st;
    ~DevFreeGuard() {
        if (*p) dev_free(*p, st);
        *p = nullptr;
    }
};
// (re)classification of a built map (rtg_map.cu); force: even when the parameters are unchanged
rtg_status classify_map(rtg_map_s* m, int variant, double k_sigma, double tau_hi, double tau_lo,
                        cudaStream_t st, bool force = false);
// planner bookkeeping (rtg_plan.cu)
cudaError_t launch_ledger(long long n, const float* prev, const float* cur, const float* wprev, float* wout,
                          cudaStream_t st);
cudaError_t launch_check_weights(long long n, const float* w, int* bad, cudaStream_t st);
cudaError_t launch_region_utility(rtg_map_s* m, const double origin[3], double size, const int dims[3], double* omega,
                                  int* count, cudaStream_t st);
cudaError_t launch_view_ring(int R, const float* cen, double d, int n, float z, rtg_traj_s* tr, cudaStream_t st);
cudaError_t launch_cost_benefit(const double* omega, const double* d, int K, void* out_dev, cudaStream_t st);
// motion-primitive tree (rtg_tree.cu), on the device; *out: candidate waypoints [K][max_depth + 1], NaN padded
rtg_status plan_tree(rtg_map_s* m, const float start[3], const float goal[2], const rtg_tree_params& p,
                     cudaStream_t st, rtg_traj_s** out, double* cost, int* n_found, int* reached,
                     long long stats[4]);

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
    // visibility records, two copies, each padded to n_gain_pad (a multiple of kTile, >= n_gain + 64)
    // with NaN means: copy A at [0, n_gain) sorted by (iy, ix, iz) -- whole columns for the flank runs;
    // copy B at [n_gain_pad, n_gain_pad + n_gain) sorted by (iy, iz, ix) -- x-contiguous z-slabs.
    // Copy B is counting-sorted from the inputs; copy A is derived from it (cell blocks moved in
    // z-fastest order).  gidx is parallel to copy B.
    long long n_gain_pad = 0;
    rtg::GRec* grec = nullptr;           // [2 * n_gain_pad]
    int* gidx = nullptr;                 // [n_gain_pad] original index per copy-B record
    int* gstartA = nullptr;              // [ncellsA + 1] first copy-A record of column (iy, ix)
    int2* zocc = nullptr;                // [ny][nxb] occupied z-cell range {lo, hi} of each row block of
                                         // kZoccX x-cells (lo > hi: empty)
    rtg::TabP* gtabP = nullptr;          // [ny][nx + 1][nz], z-fastest: entry (iy, ix, iz) = the first copy-B
                                         // record (relative to n_gain_pad) of cell (iy, iz, ix) (ix = nx: end
                                         // of the z-slab) and the exclusive prefixes there (packed, TabP)
    rtg::GainGrid gg{};
    // collision records (sorted by collision cell), padded likewise
    long long n_col_pad = 0;
    rtg::CRec* crec = nullptr;
    rtg::CMat* cmat = nullptr;
    rtg::CSrc* csrc = nullptr;           // the fp32 inputs of each collision record (FP64 re-decisions)
    int* cstart = nullptr;               // [ncells+1]
    rtg::ColGrid cg{};
    float rb_max = 0.f;
    float gq = 0.f;                      // FP32 collision guard
    double gq64 = 0.0;                   // (the same before rounding: the collision records' radius margin)
    // layout maps (rtg_map_create_layout): grids and capacity fixed at creation, rebuilt from new data
    // without a host synchronisation (rtg_map_rebuild); n_gain / n_col then hold the capacity until
    // rtg_map_check reads the counts of the last rebuild, which stay on the device with its validation
    bool layout = false;
    long long cap = 0;
    rtg_map_layout lay{};
    void* dbounds = nullptr;             // device: validation flags, counts and bounds of the last rebuild
    // classification
    rtg::ClassState* cls = nullptr;      // device
    double* red_scratch = nullptr;       // device partials for the FP64 reductions
    int cls_variant = -1;
    double cls_k = 0, cls_th = 0, cls_tl = 0;
    bool cls_th_nan = true, cls_tl_nan = true;
    long long bytes = 0;
    std::vector<void*> allocs;
};

// the shared start state as a one-waypoint info list (rtg_score with RTG_SCORE_INCLUDE_START)
struct StartState {
    float pose[4];             // x, y, z, yaw
    long long gq;              // exact fixed-point gain sum of the start's view
    int nh, nl;                // visible H / L counts
    int list[1], count[1], counter[1], pad[1];
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
    bool borrowed = false;   // rtg_traj_wrap: the arrays belong to the caller
    bool has_start = false;  // shared start state x_i(0) (rtg_traj_set_start, samplers)
    float start[4] = {0.f, 0.f, 0.f, 0.f};
};
