// rtg_api.cu -- the extern "C" boundary of librtg (include/rtg.h): argument validation,
// handle ownership, host<->device staging and launch orchestration.  No compute happens
// here; every step of the path runs in the kernels of rtg_map.cu / rtg_score.cu.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <vector>
#include <cstring>
#include <mutex>
#include <new>
#include <string>

#include "rtg_host.hpp"

namespace rtg {

static thread_local std::string g_last_error;

void set_error(const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
}

// ------------------------------------------------------------------ launch accounting / profiling
static std::atomic<long long> g_launches{0};
static std::atomic<bool> g_prof_on{false};
struct ProfRec {
    int phase;
    cudaEvent_t a, b;
};
static std::mutex g_prof_mu;
static std::vector<ProfRec> g_prof;
static std::vector<cudaEvent_t> g_prof_pending_begin[8];

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void prof_begin(int phase, cudaStream_t st) {
    if (!g_prof_on.load(std::memory_order_relaxed)) return;
    cudaEvent_t a;
    if (cudaEventCreate(&a) != cudaSuccess) return;
    cudaEventRecord(a, st);
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof_pending_begin[phase & 7].push_back(a);
}

void prof_end(int phase, cudaStream_t st) {
    if (!g_prof_on.load(std::memory_order_relaxed)) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    auto& pend = g_prof_pending_begin[phase & 7];
    if (pend.empty()) return;
    cudaEvent_t a = pend.back();
    pend.pop_back();
    cudaEvent_t b;
    if (cudaEventCreate(&b) != cudaSuccess) return;
    cudaEventRecord(b, st);
    g_prof.push_back(ProfRec{phase & 7, a, b});
}

static std::mutex g_pool_mu;
static bool g_pool_ready[64] = {false};

static void ensure_pool(int dev) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    if (dev < 0 || dev >= 64 || g_pool_ready[dev]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    g_pool_ready[dev] = true;
}

cudaError_t dev_alloc(void** p, size_t bytes, cudaStream_t st) {
    return cudaMallocAsync(p, bytes > 0 ? bytes : 16, st);
}
void dev_free(void* p, cudaStream_t st) {
    if (p) cudaFreeAsync(p, st);
}


// defined in rtg_map.cu / rtg_score.cu
rtg_status create_layout_map(rtg_map_s* m, const rtg_map_layout* L, const rtg_map_options* opt, cudaStream_t st);
rtg_status rebuild_map(rtg_map_s* m, long long n, const float* means, const float* quats, const float* scales,
                       const float* opacity, const float* w, const unsigned char* flags, cudaStream_t st);
rtg_status check_layout_map(rtg_map_s* m, cudaStream_t st);
rtg_status build_map(rtg_map_s* m, const float* means, const float* quats, const float* scales, const float* opacity,
                     const float* w, const unsigned char* flags, const rtg_map_options* opt, cudaStream_t st);
CamK make_cam(const rtg_camera& c, const double* cam64_dev);
cudaError_t launch_phase_a(rtg_map_s* m, rtg_traj_s* tr, int mode, int* first_col, unsigned char* wp_col, int all_wp,
                           int* counter, unsigned long long* stats, cudaStream_t st);
cudaError_t launch_list(const int* first_col, int K, int T, int stride, int full_gain, int* list, int* count,
                        int* ranked, cudaStream_t st);
cudaError_t launch_iota(int* list, long long n, int* count, cudaStream_t st);
cudaError_t launch_phase_b(rtg_map_s* m, rtg_traj_s* tr, int mode, const CamK& cam, const int* list,
                           const int* count, long long list_max, long long* wp_gq, int* wp_nh, int* wp_nl,
                           int* counter, unsigned long long* stats, cudaStream_t st);
cudaError_t launch_reduce(rtg_map_s* m, rtg_traj_s* tr, const rtg_score_params& p, const int* first_col,
                          const long long* wp_gq, const int* wp_nh, const int* wp_nl, const StartState* start, int* out_first,
                          unsigned char* out_feasible, double* out_gain, double* out_util, cudaStream_t st);
cudaError_t launch_start_setup(const float pose[4], StartState* st_dev, cudaStream_t st);
cudaError_t launch_debug_wp(long long n, const long long* wp_gq, const ClassState* cs, double* out, cudaStream_t st);
cudaError_t launch_pair_mask(rtg_map_s* m, rtg_traj_s* tr, unsigned* mask, cudaStream_t st);
cudaError_t launch_best(const double* u, int K, long long base, void* out_dev, cudaStream_t st);
cudaError_t launch_set_cam64(const rtg_camera& c, double* dst, cudaStream_t st);
cudaError_t launch_sampler_di(int K, int T, double dt, const float* start, const float* v0, const float* ax,
                              const float* ay, rtg_traj_s* tr, cudaStream_t st);
cudaError_t launch_sampler(int K, int T, double dt, const float* start, const float* v, const float* om,
                           rtg_traj_s* tr, cudaStream_t st);

__global__ void k_fill_int(int* p, long long n, int v) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

}  // namespace rtg

using namespace rtg;

namespace {

rtg_status invalid(const char* msg) {
    set_error("%s", msg);
    return RTG_ERR_INVALID_ARGUMENT;
}

// converts a CUDA error; a sticky error poisons the given handle flag
rtg_status cuda_fail(cudaError_t e, const char* where, bool* poison) {
    set_error("%s: %s", where, cudaGetErrorString(e));
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        return RTG_ERR_OUT_OF_MEMORY;
    }
    // sticky errors cannot be cleared; the context is unusable
    cudaError_t again = cudaGetLastError();
    (void)again;
    if (poison && cudaDeviceSynchronize() != cudaSuccess) *poison = true;
    return RTG_ERR_CUDA;
}

#define API_CK(expr, poison)                                      \
    do {                                                          \
        cudaError_t e_ = (expr);                                  \
        if (e_ != cudaSuccess) return cuda_fail(e_, #expr, poison); \
    } while (0)

bool finite_f(float v) { return std::isfinite(v); }

rtg_status check_camera(const rtg_camera* c) {
    if (!c) return invalid("camera is NULL");
    if (c->width <= 0 || c->height <= 0) return invalid("camera width/height must be > 0");
    if (!(c->fx > 0) || !(c->fy > 0) || !finite_f(c->fx) || !finite_f(c->fy)) return invalid("camera fx, fy must be finite and > 0");
    if (!(c->cx >= 0 && c->cx <= c->width) || !(c->cy >= 0 && c->cy <= c->height))
        return invalid("camera principal point must satisfy 0 <= cx <= width, 0 <= cy <= height");
    if (!(c->z_near >= 0) || !(c->z_far > c->z_near) || !finite_f(c->z_far))
        return invalid("camera depth range must satisfy 0 <= z_near < z_far < inf");
    return RTG_OK;
}

rtg_status check_params(const rtg_score_params* p) {
    if (!p) return invalid("params is NULL");
    if (!(p->lambda_xi >= 0) || !finite_f(p->lambda_xi)) return invalid("lambda_xi must be finite and >= 0");
    if (!(p->k_sigma >= 0) || !finite_f(p->k_sigma)) return invalid("k_sigma must be finite and >= 0");
    if (p->variant < RTG_VARIANT_XI || p->variant > RTG_VARIANT_SQ) return invalid("unknown variant");
    if (p->info_stride < 1) return invalid("info_stride must be >= 1");
    if (p->mode != RTG_MODE_DENSE && p->mode != RTG_MODE_CULLED) return invalid("unknown mode");
    if (p->flags & ~(unsigned)(RTG_SCORE_FULL_GAIN | RTG_SCORE_NO_COLLISION | RTG_SCORE_INCLUDE_START))
        return invalid("unknown flag bits");
    if (std::isinf(p->tau_hi) || std::isinf(p->tau_lo)) return invalid("tau must be finite or NaN");
    return RTG_OK;
}

rtg_status check_map(rtg_map m) {
    if (!m) return invalid("map handle is NULL");
    if (m->poisoned) {
        set_error("map handle poisoned by an earlier CUDA error");
        return RTG_ERR_BAD_HANDLE;
    }
    return RTG_OK;
}

rtg_status check_traj(rtg_traj t) {
    if (!t) return invalid("trajectory handle is NULL");
    if (t->poisoned) {
        set_error("trajectory handle poisoned by an earlier CUDA error");
        return RTG_ERR_BAD_HANDLE;
    }
    return RTG_OK;
}

template <typename T>
cudaError_t stage(const T* src, size_t count, rtg_mem kind, T** dst_dev, cudaStream_t st) {
    // returns a device pointer to the data: a staged copy for host input, the pointer itself otherwise
    if (kind == RTG_MEM_DEVICE || src == nullptr) {
        *dst_dev = const_cast<T*>(src);
        return cudaSuccess;
    }
    cudaError_t e = dev_alloc((void**)dst_dev, sizeof(T) * (count ? count : 1), st);
    if (e != cudaSuccess) return e;
    if (count) e = cudaMemcpyAsync(*dst_dev, src, sizeof(T) * count, cudaMemcpyHostToDevice, st);
    return e;
}

}  // namespace

extern "C" {

const char* rtg_status_string(rtg_status s) {
    switch (s) {
        case RTG_OK: return "RTG_OK";
        case RTG_ERR_INVALID_ARGUMENT: return "RTG_ERR_INVALID_ARGUMENT";
        case RTG_ERR_CUDA: return "RTG_ERR_CUDA";
        case RTG_ERR_OUT_OF_MEMORY: return "RTG_ERR_OUT_OF_MEMORY";
        case RTG_ERR_NO_FEASIBLE: return "RTG_ERR_NO_FEASIBLE";
        case RTG_ERR_BAD_HANDLE: return "RTG_ERR_BAD_HANDLE";
    }
    return "RTG_ERR_UNKNOWN";
}

const char* rtg_last_error(void) { return g_last_error.c_str(); }

const char* rtg_version(void) { return "rtg 0.1 sm_100a"; }

rtg_status rtg_profile_enable(int on) {
    g_prof_on.store(on != 0);
    return RTG_OK;
}

rtg_status rtg_profile_read(rtg_profile_t* out, int reset) {
    if (!out) return invalid("out is NULL");
    std::memset(out, 0, sizeof(*out));
    std::lock_guard<std::mutex> lk(g_prof_mu);
    for (auto& r : g_prof) {
        float ms = 0.f;
        if (cudaEventSynchronize(r.b) == cudaSuccess && cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess) {
            out->ms[r.phase] += ms;
            out->calls[r.phase] += 1;
        }
    }
    out->launches = g_launches.load();
    if (reset) {
        for (auto& r : g_prof) {
            cudaEventDestroy(r.a);
            cudaEventDestroy(r.b);
        }
        g_prof.clear();
        g_launches.store(0);
    }
    cudaGetLastError();
    return RTG_OK;
}

rtg_status rtg_map_create_ex(int device, long long n, rtg_mem kind, const float* means, const float* quats,
                             const float* scales, const float* opacity, const float* info_w,
                             const unsigned char* flags, const rtg_robot* robot, const rtg_map_options* opts,
                             void* stream, rtg_map* out) {
    if (!out) return invalid("out is NULL");
    *out = nullptr;
    // two padded record copies are indexed with 32-bit integers
    if (n < 0 || n >= (1LL << 30) - 4096) return invalid("n must satisfy 0 <= n < 2^30 - 4096");
    if (kind != RTG_MEM_HOST && kind != RTG_MEM_DEVICE) return invalid("unknown memory kind");
    if (n > 0 && (!means || !quats || !scales || !info_w)) return invalid("means, quats, scales and info_w are required");
    if (!robot) return invalid("robot is NULL");
    if (!(robot->r_robot >= 0) || !finite_f(robot->r_robot)) return invalid("r_robot must be finite and >= 0");
    if (!(robot->lambda_g > 0) || !finite_f(robot->lambda_g)) return invalid("lambda_g must be finite and > 0");
    if (robot->collide_rule != RTG_COLLIDE_ELLIPSOID && robot->collide_rule != RTG_COLLIDE_PRINCIPAL_AXIS)
        return invalid("unknown collide_rule");
    if (opts && (!std::isfinite(opts->gain_cell_xy) || !std::isfinite(opts->gain_cell_z) || !std::isfinite(opts->col_cell) ||
                 !std::isfinite(opts->gain_cell_x) || (opts->gain_z_centred && !std::isfinite(opts->gain_z_centre))))
        return invalid("grid options must be finite");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
        cudaGetLastError();
        return invalid("invalid device ordinal (no CUDA device?)");
    }
    API_CK(cudaSetDevice(device), nullptr);
    ensure_pool(device);
    cudaStream_t st = (cudaStream_t)stream;
    rtg_map_s* m = new (std::nothrow) rtg_map_s();
    if (!m) return RTG_ERR_OUT_OF_MEMORY;
    m->device = device;
    m->stream = st;
    m->n = n;
    m->robot = *robot;
    const float *dm = nullptr, *dq = nullptr, *ds = nullptr, *dop = nullptr, *dw = nullptr;
    const unsigned char* df = nullptr;
    cudaError_t e = stage(means, 3 * (size_t)n, kind, (float**)&dm, st);
    if (e == cudaSuccess) e = stage(quats, 4 * (size_t)n, kind, (float**)&dq, st);
    if (e == cudaSuccess) e = stage(scales, 3 * (size_t)n, kind, (float**)&ds, st);
    if (e == cudaSuccess) e = stage(opacity, (size_t)n, kind, (float**)&dop, st);
    if (e == cudaSuccess) e = stage(info_w, (size_t)n, kind, (float**)&dw, st);
    if (e == cudaSuccess) e = stage(flags, (size_t)n, kind, (unsigned char**)&df, st);
    rtg_status s;
    if (e != cudaSuccess) {
        s = cuda_fail(e, "rtg_map_create staging", nullptr);
    } else {
        prof_begin(PH_MAP, st);
        s = build_map(m, dm, dq, ds, dop, dw, df, opts, st);
        prof_end(PH_MAP, st);
    }
    if (kind == RTG_MEM_HOST) {
        dev_free((void*)dm, st); dev_free((void*)dq, st); dev_free((void*)ds, st);
        dev_free((void*)dop, st); dev_free((void*)dw, st); dev_free((void*)df, st);
    }
    if (s != RTG_OK) {
        for (void* p : m->allocs) dev_free(p, st);
        delete m;
        return s;
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) {
        for (void* p : m->allocs) dev_free(p, st);
        delete m;
        return cuda_fail(e, "rtg_map_create", nullptr);
    }
    *out = m;
    return RTG_OK;
}

rtg_status rtg_map_create(int device, long long n, rtg_mem kind, const float* means, const float* quats,
                          const float* scales, const float* opacity, const float* info_w, const unsigned char* flags,
                          const rtg_robot* robot, void* stream, rtg_map* out) {
    return rtg_map_create_ex(device, n, kind, means, quats, scales, opacity, info_w, flags, robot, nullptr, stream,
                             out);
}

static rtg_status check_robot_opts(const rtg_robot* robot, const rtg_map_options* opts) {
    if (!robot) return invalid("robot is NULL");
    if (!(robot->r_robot >= 0) || !finite_f(robot->r_robot)) return invalid("r_robot must be finite and >= 0");
    if (!(robot->lambda_g > 0) || !finite_f(robot->lambda_g)) return invalid("lambda_g must be finite and > 0");
    if (robot->collide_rule != RTG_COLLIDE_ELLIPSOID && robot->collide_rule != RTG_COLLIDE_PRINCIPAL_AXIS)
        return invalid("unknown collide_rule");
    if (opts && (!std::isfinite(opts->gain_cell_xy) || !std::isfinite(opts->gain_cell_z) || !std::isfinite(opts->col_cell) ||
                 !std::isfinite(opts->gain_cell_x) || (opts->gain_z_centred && !std::isfinite(opts->gain_z_centre))))
        return invalid("grid options must be finite");
    return RTG_OK;
}

rtg_status rtg_map_create_layout(int device, const rtg_map_layout* layout, const rtg_robot* robot,
                                 const rtg_map_options* opts, void* stream, rtg_map* out) {
    if (!out) return invalid("out is NULL");
    *out = nullptr;
    if (!layout) return invalid("layout is NULL");
    const rtg_map_layout& L = *layout;
    if (L.capacity < 1 || L.capacity >= (1LL << 30) - 4096) return invalid("capacity must satisfy 1 <= capacity < 2^30 - 4096");
    for (int d = 0; d < 3; ++d)
        if (!finite_f(L.gain_lo[d]) || !finite_f(L.gain_hi[d]) || !(L.gain_lo[d] <= L.gain_hi[d]) ||
            !finite_f(L.col_lo[d]) || !finite_f(L.col_hi[d]) || !(L.col_lo[d] <= L.col_hi[d]))
            return invalid("layout boxes must be finite with lo <= hi");
    if (!(L.rb_max > 0) || !finite_f(L.rb_max)) return invalid("layout rb_max must be finite and > 0");
    if (!(L.rho_max >= 1) || !finite_f(L.rho_max)) return invalid("layout rho_max must be finite and >= 1");
    rtg_status s = check_robot_opts(robot, opts);
    if (s != RTG_OK) return s;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
        cudaGetLastError();
        return invalid("invalid device ordinal (no CUDA device?)");
    }
    API_CK(cudaSetDevice(device), nullptr);
    ensure_pool(device);
    cudaStream_t st = (cudaStream_t)stream;
    rtg_map_s* m = new (std::nothrow) rtg_map_s();
    if (!m) return RTG_ERR_OUT_OF_MEMORY;
    m->device = device;
    m->stream = st;
    m->robot = *robot;
    s = create_layout_map(m, layout, opts, st);
    cudaError_t e = s == RTG_OK ? cudaGetLastError() : cudaSuccess;
    if (s == RTG_OK && e != cudaSuccess) s = cuda_fail(e, "rtg_map_create_layout", nullptr);
    if (s != RTG_OK) {
        for (void* p : m->allocs) dev_free(p, st);
        delete m;
        return s;
    }
    *out = m;
    return RTG_OK;
}

rtg_status rtg_map_rebuild(rtg_map m, long long n, const float* means, const float* quats, const float* scales,
                           const float* opacity, const float* info_w, const unsigned char* flags, void* stream) {
    rtg_status s = check_map(m);
    if (s != RTG_OK) return s;
    if (!m->layout) return invalid("rtg_map_rebuild needs a map from rtg_map_create_layout");
    if (n < 0 || n > m->cap) return invalid("n must satisfy 0 <= n <= the layout's capacity");
    if (n > 0 && (!means || !quats || !scales || !info_w)) return invalid("means, quats, scales and info_w are required");
    API_CK(cudaSetDevice(m->device), nullptr);
    cudaStream_t st = (cudaStream_t)stream;
    prof_begin(PH_MAP, st);
    s = rebuild_map(m, n, means, quats, scales, opacity, info_w, flags, st);
    prof_end(PH_MAP, st);
    if (s != RTG_OK) return s;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "rtg_map_rebuild", &m->poisoned);
    return RTG_OK;
}

rtg_status rtg_map_check(rtg_map m, void* stream) {
    rtg_status s = check_map(m);
    if (s != RTG_OK) return s;
    if (!m->layout) return RTG_OK;   // rtg_map_create validated its data before returning
    API_CK(cudaSetDevice(m->device), nullptr);
    return check_layout_map(m, (cudaStream_t)stream);
}

rtg_status rtg_map_destroy(rtg_map m) {
    if (!m) return invalid("map handle is NULL");
    cudaSetDevice(m->device);
    for (void* p : m->allocs) dev_free(p, m->stream);
    delete m;
    return RTG_OK;
}

rtg_status rtg_map_info(rtg_map m, rtg_map_info_t* out) {
    rtg_status s = check_map(m);
    if (s != RTG_OK) return s;
    if (!out) return invalid("out is NULL");
    cudaSetDevice(m->device);
    if (m->layout) {   // the counts of the last rebuild (and its validation)
        s = check_layout_map(m, m->stream);
        if (s != RTG_OK) return s;
    }
    ClassState cs;
    cudaError_t e = cudaMemcpyAsync(&cs, m->cls, sizeof(cs), cudaMemcpyDeviceToHost, m->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(m->stream);
    if (e != cudaSuccess) return cuda_fail(e, "rtg_map_info", &m->poisoned);
    out->n = m->n;
    out->n_collide = m->n_col;
    out->n_gain = m->n_gain;
    out->tau_hi = cs.tau_hi;
    out->tau_lo = cs.tau_lo;
    out->u_mean = cs.mean;
    out->u_std = cs.std;
    out->fixed_point_shift = cs.shift;
    out->gain_dims[0] = m->gg.nx; out->gain_dims[1] = m->gg.ny; out->gain_dims[2] = m->gg.nz;
    out->col_dims[0] = m->cg.nx; out->col_dims[1] = m->cg.ny; out->col_dims[2] = m->cg.nz;
    out->rb_max = m->rb_max;
    out->device_bytes = m->bytes;
    return RTG_OK;
}

static rtg_status traj_alloc(int device, int K, int T, cudaStream_t st, rtg_traj* out, rtg_traj_s** res) {
    if (!out) return invalid("out is NULL");
    *out = nullptr;
    if (K < 1 || T < 1 || (long long)K * T >= (1LL << 31)) return invalid("need K >= 1, T >= 1, K*T < 2^31");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
        cudaGetLastError();
        return invalid("invalid device ordinal (no CUDA device?)");
    }
    API_CK(cudaSetDevice(device), nullptr);
    ensure_pool(device);
    rtg_traj_s* t = new (std::nothrow) rtg_traj_s();
    if (!t) return RTG_ERR_OUT_OF_MEMORY;
    t->device = device;
    t->stream = st;
    t->K = K;
    t->T = T;
    size_t n = (size_t)K * T;
    float* base = nullptr;
    cudaError_t e = dev_alloc((void**)&base, sizeof(float) * 4 * n, st);
    if (e != cudaSuccess) {
        delete t;
        return cuda_fail(e, "rtg_traj alloc", nullptr);
    }
    t->x = base;
    t->y = base + n;
    t->z = base + 2 * n;
    t->yaw = base + 3 * n;
    *res = t;
    return RTG_OK;
}

rtg_status rtg_traj_upload(int device, int K, int T, rtg_mem kind, const float* x, const float* y, const float* z,
                           const float* yaw, void* stream, rtg_traj* out) {
    if (!x || !y || !z || !yaw) return invalid("x, y, z and yaw are required");
    if (kind != RTG_MEM_HOST && kind != RTG_MEM_DEVICE) return invalid("unknown memory kind");
    cudaStream_t st = (cudaStream_t)stream;
    rtg_traj_s* t = nullptr;
    rtg_status s = traj_alloc(device, K, T, st, out, &t);
    if (s != RTG_OK) return s;
    size_t bytes = sizeof(float) * (size_t)K * T;
    cudaMemcpyKind ck = kind == RTG_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    cudaError_t e = cudaMemcpyAsync(t->x, x, bytes, ck, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(t->y, y, bytes, ck, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(t->z, z, bytes, ck, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(t->yaw, yaw, bytes, ck, st);
    if (e != cudaSuccess) {
        dev_free(t->x, st);
        delete t;
        return cuda_fail(e, "rtg_traj_upload", nullptr);
    }
    *out = t;
    return RTG_OK;
}

rtg_status rtg_traj_sample_unicycle(int device, int K, int T, float dt, const float start[4], const float* v,
                                    const float* omega, rtg_mem kind, void* stream, rtg_traj* out) {
    if (!start || !v || !omega) return invalid("start, v and omega are required");
    if (kind != RTG_MEM_HOST && kind != RTG_MEM_DEVICE) return invalid("unknown memory kind");
    if (!(dt >= 0) || !finite_f(dt)) return invalid("dt must be finite and >= 0");
    for (int i = 0; i < 4; ++i)
        if (!finite_f(start[i])) return invalid("start state must be finite");
    cudaStream_t st = (cudaStream_t)stream;
    rtg_traj_s* t = nullptr;
    rtg_status s = traj_alloc(device, K, T, st, out, &t);
    if (s != RTG_OK) return s;
    float *dv = nullptr, *dw = nullptr;
    cudaError_t e = stage(v, (size_t)K, kind, &dv, st);
    if (e == cudaSuccess) e = stage(omega, (size_t)K, kind, &dw, st);
    if (e == cudaSuccess) e = launch_sampler(K, T, (double)dt, start, dv, dw, t, st);
    if (kind == RTG_MEM_HOST) {
        dev_free(dv, st);
        dev_free(dw, st);
    }
    if (e != cudaSuccess) {
        dev_free(t->x, st);
        delete t;
        return cuda_fail(e, "rtg_traj_sample_unicycle", nullptr);
    }
    for (int i = 0; i < 4; ++i) t->start[i] = start[i];
    t->has_start = true;
    *out = t;
    return RTG_OK;
}

rtg_status rtg_traj_sample_double_integrator(int device, int K, int T, float dt, const float start[3],
                                             const float v0[2], const float* ax, const float* ay, rtg_mem kind,
                                             void* stream, rtg_traj* out) {
    if (!start || !v0 || !ax || !ay) return invalid("start, v0, ax and ay are required");
    if (kind != RTG_MEM_HOST && kind != RTG_MEM_DEVICE) return invalid("unknown memory kind");
    if (!(dt >= 0) || !finite_f(dt)) return invalid("dt must be finite and >= 0");
    for (int i = 0; i < 3; ++i)
        if (!finite_f(start[i])) return invalid("start state must be finite");
    if (!finite_f(v0[0]) || !finite_f(v0[1])) return invalid("v0 must be finite");
    cudaStream_t st = (cudaStream_t)stream;
    rtg_traj_s* t = nullptr;
    rtg_status s = traj_alloc(device, K, T, st, out, &t);
    if (s != RTG_OK) return s;
    float *dax = nullptr, *day = nullptr;
    cudaError_t e = stage(ax, (size_t)K, kind, &dax, st);
    if (e == cudaSuccess) e = stage(ay, (size_t)K, kind, &day, st);
    if (e == cudaSuccess) e = launch_sampler_di(K, T, (double)dt, start, v0, dax, day, t, st);
    if (kind == RTG_MEM_HOST) {
        dev_free(dax, st);
        dev_free(day, st);
    }
    if (e != cudaSuccess) {
        dev_free(t->x, st);
        delete t;
        return cuda_fail(e, "rtg_traj_sample_double_integrator", nullptr);
    }
    for (int i = 0; i < 3; ++i) t->start[i] = start[i];
    t->start[3] = (v0[0] == 0.f && v0[1] == 0.f) ? 0.f : (float)std::atan2((double)v0[1], (double)v0[0]);
    t->has_start = true;
    *out = t;
    return RTG_OK;
}

rtg_status rtg_traj_set_start(rtg_traj t, const float start[4]) {
    rtg_status s = check_traj(t);
    if (s != RTG_OK) return s;
    if (!start) return invalid("start is NULL");
    for (int i = 0; i < 4; ++i)
        if (!finite_f(start[i])) return invalid("start state must be finite");
    for (int i = 0; i < 4; ++i) t->start[i] = start[i];
    t->has_start = true;
    return RTG_OK;
}

rtg_status rtg_traj_read(rtg_traj t, float* x, float* y, float* z, float* yaw, void* stream) {
    rtg_status s = check_traj(t);
    if (s != RTG_OK) return s;
    if (!x || !y || !z || !yaw) return invalid("x, y, z and yaw are required");
    cudaSetDevice(t->device);
    cudaStream_t st = (cudaStream_t)stream;
    size_t bytes = sizeof(float) * (size_t)t->K * t->T;
    API_CK(cudaMemcpyAsync(x, t->x, bytes, cudaMemcpyDeviceToDevice, st), &t->poisoned);
    API_CK(cudaMemcpyAsync(y, t->y, bytes, cudaMemcpyDeviceToDevice, st), &t->poisoned);
    API_CK(cudaMemcpyAsync(z, t->z, bytes, cudaMemcpyDeviceToDevice, st), &t->poisoned);
    API_CK(cudaMemcpyAsync(yaw, t->yaw, bytes, cudaMemcpyDeviceToDevice, st), &t->poisoned);
    return RTG_OK;
}

static bool is_device_ptr(const void* p, int device) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) && a.device == device;
}

rtg_status rtg_traj_wrap(int device, int K, int T, const float* x, const float* y, const float* z, const float* yaw,
                         rtg_traj* out) {
    if (!out) return invalid("out is NULL");
    *out = nullptr;
    if (!x || !y || !z || !yaw) return invalid("x, y, z and yaw are required");
    if (K < 1 || T < 1 || (long long)K * T >= (1LL << 31)) return invalid("need K >= 1, T >= 1, K*T < 2^31");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
        cudaGetLastError();
        return invalid("invalid device ordinal (no CUDA device?)");
    }
    if (!is_device_ptr(x, device) || !is_device_ptr(y, device) || !is_device_ptr(z, device) ||
        !is_device_ptr(yaw, device))
        return invalid("rtg_traj_wrap needs device arrays on the handle's device");
    rtg_traj_s* t = new (std::nothrow) rtg_traj_s();
    if (!t) return RTG_ERR_OUT_OF_MEMORY;
    t->device = device;
    t->K = K;
    t->T = T;
    t->x = const_cast<float*>(x);
    t->y = const_cast<float*>(y);
    t->z = const_cast<float*>(z);
    t->yaw = const_cast<float*>(yaw);
    t->borrowed = true;
    *out = t;
    return RTG_OK;
}

rtg_status rtg_traj_destroy(rtg_traj t) {
    if (!t) return invalid("trajectory handle is NULL");
    cudaSetDevice(t->device);
    if (!t->borrowed) dev_free(t->x, t->stream);
    delete t;
    return RTG_OK;
}

// scratch of one scoring pass
struct Scratch {
    int* first_col = nullptr;
    long long* wp_gq = nullptr;
    int* wp_nh = nullptr;
    int* wp_nl = nullptr;
    int* list = nullptr;
    int* ints = nullptr;                  // [0] list count, [1] phase-A counter, [2] phase-B counter
    double* cam64 = nullptr;              // FP64 camera for the re-decision branch
    int* ranked = nullptr;                // computed trajectories in order (info list build)
    unsigned long long* stats = nullptr;  // RTG_DEBUG_STATS counters (rtg_score_debug)
    StartState* start = nullptr;          // the shared start state as a 1-waypoint list (INCLUDE_START)
    void* block = nullptr;
};

static cudaError_t scratch_alloc(Scratch& s, long long K, long long T, long long list_max, const rtg_camera* cam,
                                 cudaStream_t st) {
    long long KT = K * T;
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    size_t o_first = 0;
    size_t o_gq = o_first + al(sizeof(int) * K);
    size_t o_nh = o_gq + al(sizeof(long long) * KT);
    size_t o_nl = o_nh + al(sizeof(int) * KT);
    size_t o_list = o_nl + al(sizeof(int) * KT);
    size_t o_ints = o_list + al(sizeof(int) * (list_max > 0 ? list_max : 1));
    size_t o_stats = o_ints + al(sizeof(int) * 8);
    size_t o_cam = o_stats + al(sizeof(unsigned long long) * RTG_DEBUG_STATS);
    size_t o_ranked = o_cam + al(sizeof(double) * 8);
    size_t o_start = o_ranked + al(sizeof(int) * K);
    size_t total = o_start + al(sizeof(StartState));
    cudaError_t e = dev_alloc(&s.block, total, st);
    if (e != cudaSuccess) return e;
    char* b = (char*)s.block;
    s.first_col = (int*)(b + o_first);
    s.wp_gq = (long long*)(b + o_gq);
    s.wp_nh = (int*)(b + o_nh);
    s.wp_nl = (int*)(b + o_nl);
    s.list = (int*)(b + o_list);
    s.ints = (int*)(b + o_ints);
    s.stats = (unsigned long long*)(b + o_stats);
    s.cam64 = (double*)(b + o_cam);
    s.ranked = (int*)(b + o_ranked);
    s.start = (StartState*)(b + o_start);
    // the FP64 camera (8 doubles) for the re-decision branch (a kernel parameter, not a host copy:
    // rtg_score enqueues device work only and can be captured into a CUDA graph)
    cudaError_t e2 = launch_set_cam64(*cam, s.cam64, st);
    if (e2 != cudaSuccess) return e2;
    return cudaMemsetAsync(b + o_ints, 0, o_stats + al(sizeof(unsigned long long) * RTG_DEBUG_STATS) - o_ints, st);
}

rtg_status rtg_score(rtg_map m, rtg_traj tr, const rtg_camera* cam, const rtg_score_params* p, int* first_col,
                     unsigned char* feasible, double* gain, double* utility, void* stream) {
    rtg_status s = check_map(m);
    if (s == RTG_OK) s = check_traj(tr);
    if (s == RTG_OK) s = check_camera(cam);
    if (s == RTG_OK) s = check_params(p);
    if (s != RTG_OK) return s;
    if (m->device != tr->device) return invalid("map and trajectories live on different devices");
    const bool with_start = (p->flags & RTG_SCORE_INCLUDE_START) != 0;
    if (with_start && !tr->has_start)
        return invalid("RTG_SCORE_INCLUDE_START needs the trajectories' start state (rtg_traj_set_start)");
    API_CK(cudaSetDevice(m->device), nullptr);
    cudaStream_t st = (cudaStream_t)stream;
    prof_begin(PH_CLASSIFY, st);
    s = classify_map(m, p->variant, p->k_sigma, p->tau_hi, p->tau_lo, st);
    prof_end(PH_CLASSIFY, st);
    if (s != RTG_OK) return s;
    const long long K = tr->K, T = tr->T;
    const long long per = T / p->info_stride;
    const long long list_max = K * per;
    Scratch sc;
    DevFreeGuard sc_guard{&sc.block, st};
    prof_begin(PH_OTHER, st);
    API_CK(scratch_alloc(sc, K, T, list_max, cam, st), &m->poisoned);
    const CamK ck = make_cam(*cam, sc.cam64);
    const int dense = p->mode == RTG_MODE_DENSE;
    const int full_gain = (p->flags & RTG_SCORE_FULL_GAIN) ? 1 : 0;
    note_launch(), k_fill_int<<<(unsigned)((K + 255) / 256), 256, 0, st>>>(sc.first_col, K, (int)T);
    if (dense) {
        API_CK(cudaMemsetAsync(sc.wp_gq, 0, sizeof(long long) * K * T, st), &m->poisoned);
        API_CK(cudaMemsetAsync(sc.wp_nh, 0, sizeof(int) * K * T, st), &m->poisoned);
        API_CK(cudaMemsetAsync(sc.wp_nl, 0, sizeof(int) * K * T, st), &m->poisoned);
    }
    prof_end(PH_OTHER, st);
    if (!(p->flags & RTG_SCORE_NO_COLLISION)) {
        prof_begin(PH_COLLISION, st);
        API_CK(launch_phase_a(m, tr, p->mode, sc.first_col, nullptr, 0, sc.ints + 1, nullptr, st), &m->poisoned);
        prof_end(PH_COLLISION, st);
    }
    if (per > 0) {
        prof_begin(PH_LIST, st);
        API_CK(launch_list(sc.first_col, (int)K, (int)T, p->info_stride, full_gain, sc.list, sc.ints, sc.ranked, st),
               &m->poisoned);
        prof_end(PH_LIST, st);
        prof_begin(PH_GAIN, st);
        API_CK(launch_phase_b(m, tr, p->mode, ck, sc.list, sc.ints, list_max, sc.wp_gq, sc.wp_nh, sc.wp_nl,
                              sc.ints + 2, nullptr, st),
               &m->poisoned);
        prof_end(PH_GAIN, st);
    }
    if (with_start) {
        // info state l = 0: the shared start scored once as a one-waypoint list, added per trajectory
        prof_begin(PH_GAIN, st);
        API_CK(launch_start_setup(tr->start, sc.start, st), &m->poisoned);
        rtg_traj_s one;
        one.device = tr->device;
        one.K = 1;
        one.T = 1;
        one.x = sc.start->pose + 0;
        one.y = sc.start->pose + 1;
        one.z = sc.start->pose + 2;
        one.yaw = sc.start->pose + 3;
        one.borrowed = true;
        API_CK(launch_phase_b(m, &one, p->mode, ck, sc.start->list, sc.start->count, 1, &sc.start->gq,
                              &sc.start->nh, &sc.start->nl, sc.start->counter, nullptr, st),
               &m->poisoned);
        prof_end(PH_GAIN, st);
    }
    rtg_score_params pp = *p;
    if (per == 0) pp.info_stride = (int)T + 1;   // no info waypoint: sums are empty
    prof_begin(PH_REDUCE, st);
    API_CK(launch_reduce(m, tr, pp, sc.first_col, sc.wp_gq, sc.wp_nh, sc.wp_nl, with_start ? sc.start : nullptr,
                         first_col, feasible, gain, utility, st),
           &m->poisoned);
    prof_end(PH_REDUCE, st);
    return RTG_OK;   // sc_guard frees the scratch block (stream-ordered)
}

rtg_status rtg_best(const double* utility, int K, long long index_base, void* stream, rtg_best_result* out) {
    if (!out) return invalid("out is NULL");
    out->score = -INFINITY;
    out->index = -1;
    if (!utility || K < 1) return invalid("utility must be a device array of K >= 1 values");
    cudaStream_t st = (cudaStream_t)stream;
    void* d = nullptr;
    API_CK(dev_alloc(&d, 16, st), nullptr);
    struct {
        double score;
        long long index;
    } h;
    {
        DevFreeGuard d_guard{&d, st};
        prof_begin(PH_BEST, st);
        API_CK(launch_best(utility, K, index_base, d, st), nullptr);
        prof_end(PH_BEST, st);
        API_CK(cudaMemcpyAsync(&h, d, 16, cudaMemcpyDeviceToHost, st), nullptr);
    }
    API_CK(cudaStreamSynchronize(st), nullptr);
    out->score = h.score;
    out->index = h.index;
    if (h.index < 0) {
        set_error("rtg_best: no feasible trajectory");
        return RTG_ERR_NO_FEASIBLE;
    }
    return RTG_OK;
}

rtg_status rtg_best_async(const double* utility, int K, long long index_base, rtg_best_result* out_device,
                          void* stream) {
    if (!out_device || ((uintptr_t)out_device & 7u)) return invalid("out_device must be an 8-byte aligned device pointer");
    if (!utility || K < 1) return invalid("utility must be a device array of K >= 1 values");
    cudaStream_t st = (cudaStream_t)stream;
    prof_begin(PH_BEST, st);
    API_CK(launch_best(utility, K, index_base, out_device, st), nullptr);
    prof_end(PH_BEST, st);
    return RTG_OK;
}

// ---------------------------------------------------------------- planner bookkeeping (N2, N4)

rtg_status rtg_ledger_update(int device, long long n, rtg_mem kind, const float* mu_prev, const float* mu_cur,
                             const float* w_prev, float* w_out, void* stream) {
    if (n < 0) return invalid("n must be >= 0");
    if (kind != RTG_MEM_HOST && kind != RTG_MEM_DEVICE) return invalid("unknown memory kind");
    if (n > 0 && (!mu_prev || !mu_cur || !w_prev || !w_out)) return invalid("mu_prev, mu_cur, w_prev, w_out required");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
        cudaGetLastError();
        return invalid("invalid device ordinal (no CUDA device?)");
    }
    API_CK(cudaSetDevice(device), nullptr);
    ensure_pool(device);
    cudaStream_t st = (cudaStream_t)stream;
    float *dp = nullptr, *dc = nullptr, *dw = nullptr;
    cudaError_t e = stage(mu_prev, 3 * (size_t)n, kind, &dp, st);
    if (e == cudaSuccess) e = stage(mu_cur, 3 * (size_t)n, kind, &dc, st);
    if (e == cudaSuccess) e = stage(w_prev, (size_t)n, kind, &dw, st);
    if (e == cudaSuccess) e = launch_ledger(n, dp, dc, dw, w_out, st);
    if (kind == RTG_MEM_HOST) {
        dev_free(dp, st);
        dev_free(dc, st);
        dev_free(dw, st);
    }
    if (e != cudaSuccess) return cuda_fail(e, "rtg_ledger_update", nullptr);
    return RTG_OK;
}

rtg_status rtg_map_update_weights(rtg_map m, rtg_mem kind, const float* info_w, void* stream) {
    rtg_status s = check_map(m);
    if (s != RTG_OK) return s;
    if (kind != RTG_MEM_HOST && kind != RTG_MEM_DEVICE) return invalid("unknown memory kind");
    if (m->n > 0 && !info_w) return invalid("info_w is NULL");
    API_CK(cudaSetDevice(m->device), nullptr);
    cudaStream_t st = (cudaStream_t)stream;
    const long long n = m->n;
    float* dw = nullptr;
    int* bad = nullptr;
    API_CK(stage(info_w, (size_t)n, kind, &dw, st), &m->poisoned);
    API_CK(dev_alloc((void**)&bad, sizeof(int), st), &m->poisoned);
    API_CK(cudaMemsetAsync(bad, 0, sizeof(int), st), &m->poisoned);
    API_CK(launch_check_weights(n, dw, bad, st), &m->poisoned);
    int hbad = 0;
    API_CK(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st), &m->poisoned);
    API_CK(cudaStreamSynchronize(st), &m->poisoned);
    dev_free(bad, st);
    if (hbad) {
        if (kind == RTG_MEM_HOST) dev_free(dw, st);
        return invalid("rtg_map_update_weights: info_w must be finite and >= 0");
    }
    if (n > 0) API_CK(cudaMemcpyAsync(m->w_orig, dw, sizeof(float) * n, cudaMemcpyDeviceToDevice, st), &m->poisoned);
    if (kind == RTG_MEM_HOST) dev_free(dw, st);
    prof_begin(PH_CLASSIFY, st);
    s = classify_map(m, m->cls_variant, m->cls_k, m->cls_th_nan ? NAN : m->cls_th, m->cls_tl_nan ? NAN : m->cls_tl, st,
                     true);
    prof_end(PH_CLASSIFY, st);
    if (s != RTG_OK) m->poisoned = true;
    return s;
}

rtg_status rtg_region_utility(rtg_map m, const double origin[3], double size, const int dims[3], double* omega,
                              int* count, void* stream) {
    rtg_status s = check_map(m);
    if (s != RTG_OK) return s;
    if (!origin || !dims || !omega || !count) return invalid("origin, dims, omega and count are required");
    if (!(size > 0) || !std::isfinite(size)) return invalid("size must be finite and > 0");
    for (int d = 0; d < 3; ++d) {
        if (dims[d] < 1) return invalid("dims must be >= 1");
        if (!std::isfinite(origin[d])) return invalid("origin must be finite");
    }
    if ((double)dims[0] * dims[1] * dims[2] >= 2147483647.0) return invalid("prod(dims) must be < 2^31");
    API_CK(cudaSetDevice(m->device), nullptr);
    cudaStream_t st = (cudaStream_t)stream;
    API_CK(launch_region_utility(m, origin, size, dims, omega, count, st), &m->poisoned);
    return RTG_OK;
}

rtg_status rtg_traj_view_ring(int device, int R, rtg_mem kind, const float* centroids, double size,
                              const rtg_camera* cam, int n, float z, void* stream, rtg_traj* out, double* view_dist) {
    if (!out) return invalid("out is NULL");
    *out = nullptr;
    if (R < 1 || n < 1 || (long long)R * n >= (1LL << 31)) return invalid("need R >= 1, n >= 1, R*n < 2^31");
    if (!centroids) return invalid("centroids is NULL");
    if (!(size > 0) || !std::isfinite(size) || !std::isfinite(z)) return invalid("size must be finite and > 0, z finite");
    if (kind != RTG_MEM_HOST && kind != RTG_MEM_DEVICE) return invalid("unknown memory kind");
    rtg_status s = check_camera(cam);
    if (s != RTG_OK) return s;
    // viewing distance: the region (edge size) fills the narrower field of view
    const double hf = std::atan((double)cam->cx / (double)cam->fx) +
                      std::atan(((double)cam->width - (double)cam->cx) / (double)cam->fx);
    const double vf = std::atan((double)cam->cy / (double)cam->fy) +
                      std::atan(((double)cam->height - (double)cam->cy) / (double)cam->fy);
    const double d = (size / 2.0) / std::tan(std::min(hf, vf) / 2.0);
    if (view_dist) *view_dist = d;
    cudaStream_t st = (cudaStream_t)stream;
    rtg_traj_s* t = nullptr;
    s = traj_alloc(device, R * n, 1, st, out, &t);
    if (s != RTG_OK) return s;
    float* dc = nullptr;
    cudaError_t e = stage(centroids, 3 * (size_t)R, kind, &dc, st);
    if (e == cudaSuccess) e = launch_view_ring(R, dc, d, n, z, t, st);
    if (kind == RTG_MEM_HOST) dev_free(dc, st);
    if (e != cudaSuccess) {
        dev_free(t->x, st);
        delete t;
        return cuda_fail(e, "rtg_traj_view_ring", nullptr);
    }
    *out = t;
    return RTG_OK;
}

rtg_status rtg_cost_benefit(const double* omega, const double* d, int K, void* stream, rtg_best_result* out) {
    if (!out) return invalid("out is NULL");
    out->score = -INFINITY;
    out->index = -1;
    if (!omega || !d || K < 1) return invalid("omega and d must be device arrays of K >= 1 values");
    cudaStream_t st = (cudaStream_t)stream;
    void* dv = nullptr;
    API_CK(dev_alloc(&dv, 16, st), nullptr);
    struct {
        double score;
        long long index;
    } h;
    {
        DevFreeGuard dv_guard{&dv, st};
        API_CK(launch_cost_benefit(omega, d, K, dv, st), nullptr);
        API_CK(cudaMemcpyAsync(&h, dv, 16, cudaMemcpyDeviceToHost, st), nullptr);
    }
    API_CK(cudaStreamSynchronize(st), nullptr);
    out->score = h.score;
    out->index = h.index;
    return RTG_OK;
}

rtg_status rtg_plan_tree(rtg_map m, const float start[3], const float goal[2], const rtg_tree_params* p,
                         void* stream, rtg_traj* out, double* cost, int* n_found, int* reached, long long* stats) {
    if (!out || !n_found || !reached) return invalid("out, n_found and reached are required");
    *out = nullptr;
    *n_found = 0;
    *reached = 0;
    rtg_status s = check_map(m);
    if (s != RTG_OK) return s;
    if (!start || !goal || !p) return invalid("start, goal and params are required");
    for (int i = 0; i < 3; ++i)
        if (!finite_f(start[i])) return invalid("start must be finite");
    if (!finite_f(goal[0]) || !finite_f(goal[1])) return invalid("goal must be finite");
    if (p->n_v < 1 || p->n_omega < 1 || !(p->v_max > 0) || !(p->omega_max >= 0) || !(p->dt > 0) ||
        !(p->lambda_t >= 0) || p->samples < 2 || p->max_depth < 1 || !(p->goal_radius >= 0) || p->beam < 1 ||
        p->n_traj < 1 || !finite_f(p->v_max) || !finite_f(p->omega_max) || !finite_f(p->dt) ||
        !finite_f(p->lambda_t) || !finite_f(p->goal_radius) || !finite_f(p->z) || !finite_f(p->lattice_xy) ||
        !finite_f(p->lattice_deg))
        return invalid("rtg_tree_params out of range");
    if ((long long)p->beam * p->n_v * p->n_omega >= (1LL << 31) / 32) return invalid("beam * controls too large");
    if ((long long)p->n_traj * (p->max_depth + 1) >= (1LL << 31)) return invalid("n_traj * (max_depth + 1) too large");
    API_CK(cudaSetDevice(m->device), nullptr);
    cudaStream_t st = (cudaStream_t)stream;
    return plan_tree(m, start, goal, *p, st, out, cost, n_found, reached, stats);
}

rtg_status rtg_score_debug(rtg_map m, rtg_traj tr, const rtg_camera* cam, const rtg_score_params* p,
                           unsigned char* wp_col, double* wp_gain, int* wp_nh, int* wp_nl, unsigned int* pair_mask,
                           long long* stats, void* stream) {
    rtg_status s = check_map(m);
    if (s == RTG_OK) s = check_traj(tr);
    if (s == RTG_OK) s = check_camera(cam);
    if (s == RTG_OK) s = check_params(p);
    if (s != RTG_OK) return s;
    if (m->device != tr->device) return invalid("map and trajectories live on different devices");
    if (!wp_col || !wp_gain || !wp_nh || !wp_nl) return invalid("wp_col, wp_gain, wp_nh, wp_nl are required");
    const long long K = tr->K, T = tr->T, KT = K * T;
    if (pair_mask && (double)KT * (double)m->n > 4294967296.0) return invalid("pair_mask needs K*T*N <= 2^32");
    API_CK(cudaSetDevice(m->device), nullptr);
    cudaStream_t st = (cudaStream_t)stream;
    s = classify_map(m, p->variant, p->k_sigma, p->tau_hi, p->tau_lo, st);
    if (s != RTG_OK) return s;
    Scratch sc;
    DevFreeGuard sc_guard{&sc.block, st};
    API_CK(scratch_alloc(sc, K, T, KT, cam, st), &m->poisoned);
    const CamK ck = make_cam(*cam, sc.cam64);
    note_launch(), k_fill_int<<<(unsigned)((K + 255) / 256), 256, 0, st>>>(sc.first_col, K, (int)T);
    API_CK(cudaMemsetAsync(wp_col, 0, KT, st), &m->poisoned);
    API_CK(cudaMemsetAsync(sc.wp_gq, 0, sizeof(long long) * KT, st), &m->poisoned);
    API_CK(cudaMemsetAsync(wp_nh, 0, sizeof(int) * KT, st), &m->poisoned);
    API_CK(cudaMemsetAsync(wp_nl, 0, sizeof(int) * KT, st), &m->poisoned);
    if (!(p->flags & RTG_SCORE_NO_COLLISION))
        API_CK(launch_phase_a(m, tr, p->mode, sc.first_col, wp_col, 1, sc.ints + 1, sc.stats, st), &m->poisoned);
    API_CK(launch_iota(sc.list, KT, sc.ints, st), &m->poisoned);
    API_CK(launch_phase_b(m, tr, p->mode, ck, sc.list, sc.ints, KT, sc.wp_gq, wp_nh, wp_nl, sc.ints + 2, sc.stats, st),
           &m->poisoned);
    API_CK(launch_debug_wp(KT, sc.wp_gq, m->cls, wp_gain, st), &m->poisoned);
    if (pair_mask) {
        size_t words = (size_t)((KT * m->n + 31) / 32);
        API_CK(cudaMemsetAsync(pair_mask, 0, sizeof(unsigned) * (words ? words : 1), st), &m->poisoned);
        API_CK(launch_pair_mask(m, tr, pair_mask, st), &m->poisoned);
    }
    unsigned long long hs[RTG_DEBUG_STATS] = {};
    API_CK(cudaMemcpyAsync(hs, sc.stats, sizeof(hs), cudaMemcpyDeviceToHost, st), &m->poisoned);
    dev_free(sc.block, st);
    sc.block = nullptr;
    API_CK(cudaStreamSynchronize(st), &m->poisoned);
    if (stats)
        for (int i = 0; i < RTG_DEBUG_STATS; ++i) stats[i] = (long long)hs[i];
    return RTG_OK;
}

}  // extern "C"
