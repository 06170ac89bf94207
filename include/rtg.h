/*
 * rtg.h -- C ABI of the B200-native RT-GuIDE trajectory-scoring library (librtg.so).
 *
 * The library implements the data-parallel hot path of the trajectory planner of
 * "RT-GuIDE: Real-Time Gaussian splatting for Information-Driven Exploration"
 * (arXiv 2409.18122, /root/reference/PAPER.md, cited as P:<line>):
 * batched scoring of K candidate trajectories of T waypoints against a map of N
 * 3D Gaussians.  For every (waypoint, Gaussian) pair it runs the collision test
 * and the binary field-of-view visibility test,
 * accumulates the trace-proxy information gain and the view utility xi
 * (Eq. equ:view_util), reduces each trajectory to a feasibility flag,
 * a gain and a utility (Eq. equ:traj_utility) and takes the argmax.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - Every function returns rtg_status; no C++ exception crosses the ABI.
 *    On failure, rtg_last_error() returns a thread-local detail message.
 *  - Arrays are plain pointers.  `kind` says whether input pointers are host
 *    memory (RTG_MEM_HOST: copied to the device inside the call, stream-ordered)
 *    or device memory of `device` (RTG_MEM_DEVICE: read in place).  Output
 *    pointers of rtg_score / rtg_score_debug are always caller-owned DEVICE
 *    buffers.  The caller keeps every input valid until the stream passes the call.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  All work is
 *    enqueued on it.  Only rtg_map_create (sizes its grids from the data),
 *    rtg_best (returns a host result) and rtg_score_debug synchronise it.
 *  - CUDA graphs: rtg_map_rebuild (layout maps), rtg_score in RTG_MODE_CULLED
 *    (when it does not reclassify) and rtg_best_async enqueue device work only
 *    (kernels, memsets and stream-ordered allocations freed within the call),
 *    so a capturing stream records the whole planning cycle; the graph keeps
 *    the handles' and arrays' device pointers, so a replay rebuilds from and
 *    scores whatever those buffers then hold.
 *  - Handles own their device memory until *_destroy.  Handles are not
 *    thread-safe; distinct handles on distinct streams are.
 *  - A CUDA error inside a call returns RTG_ERR_CUDA; if the error is sticky
 *    the handle is poisoned and later calls on it return RTG_ERR_BAD_HANDLE.
 *  - Arithmetic: pair tests in FP32 with an FP64 re-decision of every pair whose
 *    FP32 test lies within a proven error guard of its threshold, so each
 *    collision / visibility decision equals the FP64 decision; gains are summed
 *    exactly in 2^-S fixed point (S chosen per map), counts in integers.
 */
#ifndef RTG_H
#define RTG_H

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    RTG_OK = 0,
    RTG_ERR_INVALID_ARGUMENT = 1,
    RTG_ERR_CUDA = 2,
    RTG_ERR_OUT_OF_MEMORY = 3,
    RTG_ERR_NO_FEASIBLE = 4,      /* rtg_best: every utility is -inf (SPEC "unreachable") */
    RTG_ERR_BAD_HANDLE = 5
} rtg_status;

typedef enum { RTG_MEM_HOST = 0, RTG_MEM_DEVICE = 1 } rtg_mem;

/* per-Gaussian flag bits (uint8 flags[N]) */
enum {
    RTG_G_NO_COLLIDE = 1u,   /* excluded from collision: ground Gaussians      */
    RTG_G_NO_GAIN = 2u       /* excluded from visibility / gain / classification           */
};

/* collision rule (rtg_robot.collide_rule) */
enum {
    RTG_COLLIDE_ELLIPSOID = 0,       /* q = sum_i ((R^T (p-mu))_i / (lambda_g s_i + r_robot))^2 < 1;
                                        reduces to |p-mu| < r_robot + lambda_g r when isotropic */
    RTG_COLLIDE_PRINCIPAL_AXIS = 1   /* |p-mu| < r_robot + lambda_g max_i s_i            */
};

/* scoring variant (rtg_score_params.variant) */
enum {
    RTG_VARIANT_XI = 0,   /* utility = sum of xi = n_H - lambda_xi n_L (Eq. equ:view_util)   */
    RTG_VARIANT_SUM = 1,  /* utility = sum of visible uncertainty (RTGuIDE-sum)            */
    RTG_VARIANT_SQ = 2    /* uncertainty u = w^2 for classes and gain (RTGuIDE-sq)         */
};

/* execution mode (rtg_score_params.mode) -- identical results, different algorithms */
enum {
    RTG_MODE_DENSE = 0,   /* every waypoint x every Gaussian ("all sampled points with all
                             Gaussians at once"), smem/TMA-staged tiles             */
    RTG_MODE_CULLED = 1   /* exact spatial culling on cell grids built by rtg_map_create  */
};

/* rtg_score_params.flags */
enum {
    RTG_SCORE_FULL_GAIN = 1u,     /* compute gain/xi for infeasible trajectories too (else NaN)  */
    RTG_SCORE_NO_COLLISION = 2u,  /* gain-only viewpoints: skip collision, all feasible          */
    RTG_SCORE_INCLUDE_START = 4u  /* the shared start state x_i(0) is info state l = 0 of every
                                     trajectory (Eq. equ:traj_utility sums l = 0..L):
                                     its gain and xi are added to every computed trajectory.  The
                                     start is the handle's (rtg_traj_set_start; the samplers set
                                     it); it is not collision-checked (it must be free) */
};

typedef struct rtg_map_s* rtg_map;
typedef struct rtg_traj_s* rtg_traj;

/* Robot: r_robot >= 0 [m]; lambda_g > 0 (3 in the paper); collide_rule above. */
typedef struct {
    float r_robot;
    float lambda_g;
    int collide_rule;
} rtg_robot;

/* Pinhole camera mounted at each waypoint, optical axis along the heading, no pitch/roll
 * (x right = (sin yaw, -cos yaw, 0), y down).  width, height > 0 [px]; fx, fy > 0 [px];
 * 0 <= cx <= width, 0 <= cy <= height; 0 <= z_near < z_far [m] (depth = camera-axis Z,
 * P:138).  A Gaussian is visible iff its mean projects inside [0,W]x[0,H] with
 * z_near <= Z <= z_far (closed bounds; no extent, no occlusion). */
typedef struct {
    int width, height;
    float fx, fy, cx, cy;
    float z_near, z_far;
} rtg_camera;

/* Scoring parameters.  lambda_xi >= 0 (1 in the paper); k_sigma >= 0 (1/2);
 * info_stride >= 1: information is evaluated at waypoints t with (t+1) % info_stride == 0
 * (1 = every waypoint; 1 s / dt reproduces the paper's segment end states);
 * tau_hi / tau_lo: NaN = derive from the map as mean +- k_sigma * population std of u over
 * the gain-eligible Gaussians, else used as given (class H iff u > tau_hi,
 * L iff u < tau_lo). */
typedef struct {
    float lambda_xi;
    float k_sigma;
    int variant;
    int info_stride;
    int mode;
    unsigned flags;
    double tau_hi;
    double tau_lo;
} rtg_score_params;

typedef struct {
    double score;        /* best utility, -inf when none is feasible */
    long long index;     /* index_base + local index, -1 when none   */
} rtg_best_result;

/* Grid options for rtg_map_create_ex / rtg_map_create_layout; any size <= 0 selects the default.
 * The visibility grid has rows of height gain_cell_xy along y, cells of width gain_cell_x along x
 * and z-cells of height gain_cell_z (the culled gain kernel tests individually only Gaussians of
 * cells that straddle the frustum, so thinner rows mean fewer tests but more rows).  The z-cells
 * start at the lowest mean unless gain_z_centred is set: then one z-cell is centred on
 * gain_z_centre, e.g. the camera height of a ground robot, whose waypoints share it.  The cell
 * holding the camera straddles the frustum's top and bottom planes out to the depth where the
 * vertical field of view spans it -- hz / (2 k) with the camera at its centre, up to hz / k at an
 * edge (k = the slope of the planes) -- so centring it minimises the near-field tests.  Results do
 * not depend on any of these options. */
typedef struct {
    float gain_cell_xy;  /* visibility grid row height (y) [m]    (default 0.3)            */
    float gain_cell_z;   /* visibility grid cell height (z) [m]   (default 1.5)            */
    float col_cell;      /* collision grid cell edge [m]          (default max(0.5, r_b/2)) */
    float gain_cell_x;   /* visibility grid cell width (x) [m]    (default gain_cell_xy/4) */
    int gain_z_centred;  /* nonzero: centre a z-cell on gain_z_centre                      */
    float gain_z_centre; /* [m], finite                                                    */
} rtg_map_options;

/* Read-only facts about a built map (rtg_map_info). */
typedef struct {
    long long n, n_collide, n_gain;
    double tau_hi, tau_lo, u_mean, u_std;   /* current classification                  */
    int fixed_point_shift;                  /* gains are exact multiples of 2^-shift    */
    int gain_dims[3];                       /* visibility grid cells (x, y, z)          */
    int col_dims[3];                        /* collision grid cells (x, y, z)           */
    float rb_max;                           /* largest collision bounding radius [m]    */
    long long device_bytes;                 /* device memory owned by the handle        */
} rtg_map_info_t;

/*
 * rtg_map_create -- map intake and packing (SURVEY §8(a) a1 + a2).
 * means [3][N] (planar x|y|z), quats [4][N] (planar w|x|y|z, any non-zero norm, normalised
 * in FP64), scales [3][N] (per-axis standard deviation, > 0), opacity [N] (in [0,1]; stored,
 * unused by scoring: planning never uses alpha), info_w [N] (the displacement-magnitude
 * uncertainty ledger, finite, >= 0), flags [N] or NULL.  N = 0 is legal.
 * Packs FP64-derived FP32 records (M = diag(1/a) R^T, bounding radius, fixed-point u),
 * classifies with the default parameters and builds the visibility and collision grids.
 * Errors: RTG_ERR_INVALID_ARGUMENT on a bad pointer/size or any invalid element
 * (non-finite value, quaternion norm < 1e-12, scale <= 0, info_w < 0, opacity outside [0,1]);
 * RTG_ERR_OUT_OF_MEMORY; RTG_ERR_CUDA.  0 <= n < 2^30 - 4096.  Synchronises `stream` once.
 */
rtg_status rtg_map_create(int device, long long n, rtg_mem kind,
                          const float* means, const float* quats, const float* scales,
                          const float* opacity, const float* info_w, const unsigned char* flags,
                          const rtg_robot* robot, void* stream, rtg_map* out);
rtg_status rtg_map_create_ex(int device, long long n, rtg_mem kind,
                             const float* means, const float* quats, const float* scales,
                             const float* opacity, const float* info_w, const unsigned char* flags,
                             const rtg_robot* robot, const rtg_map_options* opts,
                             void* stream, rtg_map* out);
rtg_status rtg_map_destroy(rtg_map map);

/*
 * Layout maps: a map whose grids and capacity are fixed at creation from caller bounds, rebuilt
 * from new data with device work only -- no host synchronisation, so a CUDA graph can capture
 * rtg_map_rebuild + rtg_score + rtg_best_async (the whole planning cycle) and replay it.
 * The grids cover the layout boxes (cell sizes as rtg_map_options); rb_max and rho_max set the
 * collision search radius and the FP32 guard (larger bounds cost time, not correctness).  Scores of
 * a rebuilt map equal those of rtg_map_create on the same data (decisions and exact sums do not
 * depend on the grid).
 */
typedef struct {
    long long capacity;  /* most Gaussians a rebuild may hold, 1 <= capacity < 2^30 - 4096      */
    float gain_lo[3];    /* box holding every gain-eligible mean of every rebuild (world, m)   */
    float gain_hi[3];
    float col_lo[3];     /* box holding every collidable mean                                   */
    float col_hi[3];
    float rb_max;        /* bound on a collidable Gaussian's largest semi-axis a = lambda_g s + r_robot */
    float rho_max;       /* bound on its a_max / a_min (>= 1)                                    */
} rtg_map_layout;

/* Allocates a layout map on `device` (an empty map until the first rebuild).  Synchronous
 * allocation; RTG_ERR_INVALID_ARGUMENT for non-finite or empty boxes, bounds out of range. */
rtg_status rtg_map_create_layout(int device, const rtg_map_layout* layout, const rtg_robot* robot,
                                 const rtg_map_options* opts, void* stream, rtg_map* out);

/* Rebuilds a layout map from n <= capacity Gaussians (DEVICE arrays as rtg_map_create's, read in
 * place; flags may be NULL) with the default classification.  Enqueues device work only
 * (capturable).  The validation of rtg_map_create plus the layout (means inside the boxes, radius and
 * anisotropy within the bounds) is recorded on the device: rtg_map_check reports it.  A rebuild
 * whose data breaks the layout gives undefined scores (memory-safe: cells clamp). */
rtg_status rtg_map_rebuild(rtg_map map, long long n, const float* means, const float* quats,
                           const float* scales, const float* opacity, const float* info_w,
                           const unsigned char* flags, void* stream);

/* Synchronises `stream` and returns RTG_ERR_INVALID_ARGUMENT (detail in rtg_last_error) if the last
 * rebuild's data was invalid or broke the layout; RTG_OK otherwise (always for rtg_map_create maps).
 * Afterwards rtg_map_info reports the rebuild's record counts. */
rtg_status rtg_map_check(rtg_map map, void* stream);
rtg_status rtg_map_info(rtg_map map, rtg_map_info_t* out);

/*
 * rtg_traj_upload -- candidate trajectories.  K >= 1, T >= 1,
 * K*T < 2^31; x, y, z, yaw each [K][T] (trajectory-major), waypoint t of trajectory k at
 * index k*T + t.  Copies into a handle-owned device SoA.  Non-finite values are padding
 * (R8): such a waypoint sees nothing, and with a non-finite position it collides with
 * nothing.
 */
rtg_status rtg_traj_upload(int device, int K, int T, rtg_mem kind,
                           const float* x, const float* y, const float* z, const float* yaw,
                           void* stream, rtg_traj* out);
/*
 * rtg_traj_sample_unicycle -- on-device motion-primitive sampler:
 * trajectory k applies the constant control (v[k], omega[k]) from start = {x, y, z, yaw};
 * waypoint t is the closed-form unicycle state at time (t+1)*dt (FP64, stored as FP32),
 * heading wrapped to (-pi, pi], z constant.  v/omega are host or device per `kind`.
 */
rtg_status rtg_traj_sample_unicycle(int device, int K, int T, float dt, const float start[4],
                                    const float* v, const float* omega, rtg_mem kind,
                                    void* stream, rtg_traj* out);
/*
 * rtg_traj_sample_double_integrator -- on-device double-integrator primitives (BASELINE.json
 * configs[2]; SURVEY §8(b) optional sampler): trajectory k accelerates at the constant
 * (ax[k], ay[k]) from start = {x, y, z} with velocity v0 = {vx, vy}; waypoint l is the closed-form
 * state at t = (l+1)*dt: p = p0 + v0 t + a t^2 / 2 (FP64, stored as FP32), z constant, heading
 * atan2(vy + ay t, vx + ax t) (0 at zero velocity).  ax / ay are host or device per `kind`.
 */
rtg_status rtg_traj_sample_double_integrator(int device, int K, int T, float dt, const float start[3],
                                             const float v0[2], const float* ax, const float* ay,
                                             rtg_mem kind, void* stream, rtg_traj* out);
/*
 * rtg_traj_wrap -- zero-copy borrow of caller DEVICE arrays x, y, z, yaw (each K*T floats,
 * trajectory-major, on `device`) as a trajectory handle.  The library only
 * reads them; the caller keeps them alive and unchanged until rtg_traj_destroy (which does not free
 * them).  Errors: RTG_ERR_INVALID_ARGUMENT (NULL or non-device pointers, K < 1, T < 1,
 * K*T >= 2^31, bad device).
 */
rtg_status rtg_traj_wrap(int device, int K, int T, const float* x, const float* y, const float* z,
                         const float* yaw, rtg_traj* out);
/*
 * rtg_traj_set_start -- the shared start state {x, y, z, yaw} (host array) of the handle's K
 * trajectories, i.e. x_i(0) of Eq. equ:traj_utility, used by rtg_score with
 * RTG_SCORE_INCLUDE_START.  rtg_traj_sample_unicycle sets it to its start, the double-integrator
 * sampler to {start, atan2(v0)} (0 at zero velocity).  Errors: RTG_ERR_INVALID_ARGUMENT (NULL or
 * non-finite start), RTG_ERR_BAD_HANDLE.
 */
rtg_status rtg_traj_set_start(rtg_traj traj, const float start[4]);
/* Copies the trajectory SoA into caller device buffers (each K*T floats). */
rtg_status rtg_traj_read(rtg_traj traj, float* x, float* y, float* z, float* yaw, void* stream);
rtg_status rtg_traj_destroy(rtg_traj traj);

/*
 * rtg_score -- the planning cycle's scoring pass.
 * Outputs (caller-owned device arrays of length K):
 *   first_col[k]  first colliding waypoint index, T if none (collision is any-reduce over
 *                 the Gaussians of each waypoint)
 *   feasible[k]   1 iff first_col[k] == T
 *   gain[k]       sum over info waypoints of the trace proxy sum_{visible} u_g (Eq. eq:nbv
 *                 with binary J); NaN for infeasible k unless RTG_SCORE_FULL_GAIN
 *   utility[k]    feasible ? sum over info waypoints of xi (XI, SQ) or gain (SUM) : -inf
 * With RTG_SCORE_INCLUDE_START the info states are the start state plus the info waypoints
 * (RTG_ERR_INVALID_ARGUMENT when the handle has no start).
 * Any output pointer may be NULL (not written).  Reclassifies the map if params ask for a
 * classification other than the current one.  Does not synchronise.
 */
rtg_status rtg_score(rtg_map map, rtg_traj traj, const rtg_camera* cam, const rtg_score_params* params,
                     int* first_col, unsigned char* feasible, double* gain, double* utility,
                     void* stream);

/*
 * rtg_best -- argmax over utility[K] (device), ties -> lowest index (SPEC S:419 reading),
 * returning index_base + k (global index when trajectories are sharded across ranks).
 * Synchronises the stream.  RTG_ERR_NO_FEASIBLE (with index -1, score -inf) when every
 * utility is -inf.
 */
rtg_status rtg_best(const double* utility, int K, long long index_base, void* stream,
                    rtg_best_result* out);

/*
 * rtg_best_async -- rtg_best without the host result: the same argmax written to
 * out_device (one rtg_best_result in caller-owned, 8-byte aligned DEVICE memory; index -1
 * and score -inf when nothing is feasible).  Does not synchronise (capturable).
 */
rtg_status rtg_best_async(const double* utility, int K, long long index_base, rtg_best_result* out_device,
                          void* stream);

/*
 * rtg_score_debug -- parity/debug: per-waypoint outputs for EVERY waypoint (no early exit,
 * every t regardless of info_stride): wp_col[K*T] (uint8 collision), wp_gain[K*T] (double),
 * wp_nh[K*T], wp_nl[K*T] (visible H / L counts), computed by the `params->mode` kernels.
 * pair_mask (or NULL): ceil(K*T*N/32) words, bit (i*N + g) = waypoint i collides with
 * Gaussian g (original index), only when K*T*N <= 2^32.  stats (host, or NULL): RTG_DEBUG_STATS
 * (= 12) counters {collision pairs FP64-redecided, visibility pairs FP64-redecided, visibility
 * pairs tested individually, (row, z-cell) x-runs added whole, collision candidates tested,
 * visibility pairs tested in the horizontally straddling flanks of rows, (row, z-cell) units cut,
 * individually tested pairs visible, footprint rows classified, tested runs (contiguous record
 * ranges queued for individual tests), 16-byte table entries loaded by the (row, z-cell) units,
 * bytes of column starts and z-occupancy blocks loaded by the footprint rows}
 * (culled mode; dense mode fills the first two).  Synchronises the stream.
 */
enum { RTG_DEBUG_STATS = 12 };
rtg_status rtg_score_debug(rtg_map map, rtg_traj traj, const rtg_camera* cam,
                           const rtg_score_params* params,
                           unsigned char* wp_col, double* wp_gain, int* wp_nh, int* wp_nl,
                           unsigned int* pair_mask, long long* stats, void* stream);

/*
 * ---------------------------------------------------------------- planner bookkeeping
 *
 * rtg_ledger_update -- N4, the uncertainty ledger: for each of n Gaussians,
 * w_out[g] = ||mu_cur[g] - mu_prev[g]||_2 (norm of the fp32 differences taken in FP64, rounded
 * to fp32) when any coordinate of the mean changed, w_prev[g] otherwise ("Gaussians that remain
 * unchanged in the most recent update retain their previously computed displacement values").
 * mu_prev, mu_cur [3][N] planar and w_prev [N] are host or device per `kind`; w_out [N] is a
 * caller-owned device array (may equal w_prev when that is on the device).  Does not synchronise.
 * Errors: RTG_ERR_INVALID_ARGUMENT (n < 0, NULL pointers, bad device).
 */
rtg_status rtg_ledger_update(int device, long long n, rtg_mem kind, const float* mu_prev, const float* mu_cur,
                             const float* w_prev, float* w_out, void* stream);

/*
 * rtg_map_update_weights -- N4: replaces the map's information weights (the ledger, [N] in the
 * map's input order, host or device per `kind`) without repacking its geometry, and reclassifies
 * the map with its current classification parameters (a2).  Synchronises the stream once
 * (validation).  Errors: RTG_ERR_INVALID_ARGUMENT on a NULL pointer or any weight that is
 * non-finite or < 0 (the map is left unchanged); RTG_ERR_BAD_HANDLE; RTG_ERR_CUDA.
 */
rtg_status rtg_map_update_weights(rtg_map map, rtg_mem kind, const float* info_w, void* stream);

/*
 * rtg_region_utility -- N2: the enclosing space is partitioned into cuboidal
 * regions of edge `size` (2.5 m in the paper) with lower corner origin[3] and dims[3]
 * regions (flat index (iz * dims[1] + iy) * dims[0] + ix); a gain-eligible Gaussian (ground plane
 * excluded) with mean mu lies in region floor((mu - origin) / size) (FP64) when that is
 * inside dims.  count[r] = M_r, omega[r] = (1/M_r) sum_{g in r} w_g (0 for an empty region).  The
 * sums are exact fixed-point integers (quantum 2^-S, S = floor(52 - log2(sum M * max w))), so the
 * result is deterministic.  omega [prod dims] (double) and count [prod dims] (int) are caller-owned
 * device arrays.  Does not synchronise.  Errors: RTG_ERR_INVALID_ARGUMENT (size <= 0, dims < 1,
 * prod dims >= 2^31), RTG_ERR_BAD_HANDLE, RTG_ERR_CUDA.
 */
rtg_status rtg_region_utility(rtg_map map, const double origin[3], double size, const int dims[3], double* omega,
                              int* count, void* stream);

/*
 * rtg_traj_view_ring -- N2 viewpoint placement: for each of R region
 * centroids (planar [3][R], host or device per `kind`), n viewpoints on the circle of radius
 * d = (size/2) / tan(min(hfov, vfov)/2) around the centroid in the plane z (hfov, vfov: the angles
 * [0, W] and [0, H] subtend at the optical centre), at angles 2 pi j / n, heading towards the
 * centroid: a trajectory handle with K = R * n, T = 1 (viewpoint v = r * n + j) that rtg_score
 * scores as gain-only views (RTG_SCORE_NO_COLLISION).  *view_dist (or NULL) receives d.
 * Errors: RTG_ERR_INVALID_ARGUMENT (R, n < 1, R * n >= 2^31, size <= 0, bad camera).
 */
rtg_status rtg_traj_view_ring(int device, int R, rtg_mem kind, const float* centroids, double size,
                              const rtg_camera* cam, int n, float z, void* stream, rtg_traj* out, double* view_dist);

/*
 * rtg_cost_benefit -- N2 guidance selection: argmax over K viewpoints of
 * omega[j] / e^{d[j]} (FP64; d = path distance to the viewpoint, omega = its utility), ties ->
 * smaller d, then smaller j.  omega, d are device arrays of K >= 1 values.  Synchronises the
 * stream.  Errors: RTG_ERR_INVALID_ARGUMENT (NULL pointers, K < 1), RTG_ERR_CUDA.
 */
rtg_status rtg_cost_benefit(const double* omega, const double* d, int K, void* stream, rtg_best_result* out);

/*
 * rtg_plan_tree -- N3, trajectory candidate generation on the device (§IV-B2):
 * a tree of unicycle motion primitives (fixed controls u = (v, w) over dt; v on a uniform grid of
 * [0, v_max] with n_v points incl. both ends ({v_max} when n_v = 1), w likewise on
 * [-omega_max, omega_max] ({0} when n_omega = 1)) is grown from start = {x, y, theta}
 * layer by layer.  Each layer expands every frontier node by every control; the `samples` states
 * at t_j = j dt / (samples - 1), j = 1 .. samples - 1 (closed form), are collision-
 * checked against the map with the a4 test at height z, all in one launch; a primitive with
 * a colliding sample is discarded.  A child costs g = g_parent + (lambda_t + v^2 + w^2) dt
 * (Eq. low_level_planner); it is dropped when its (lattice_xy, lattice_xy, lattice_deg) lattice cell
 * was already reached with a cost <= g (lattice_xy <= 0: no lattice); it is a candidate (not
 * expanded) when ||p - goal|| <= goal_radius.  The next frontier keeps the `beam` children of
 * lowest f = g + ||goal - p|| / v_max.  After max_depth layers the n_traj cheapest
 * candidates are returned (*reached = 1), or, when none reached the goal, the n_traj nodes closest
 * to it (*reached = 0).  Ties always go to creation order (node, then control).
 * *out: trajectory handle with K = *n_found (<= n_traj), T = max_depth + 1, waypoint l = the
 * state after l primitives (l = 0: start; NaN after the candidate's last primitive); cost (host,
 * n_traj entries or NULL) receives the candidates' g; stats (host long long[4] or NULL):
 * nodes expanded, nodes created, samples checked (a primitive's samples are tested together, so
 * every sample of an expanded primitive counts), collision candidates tested.  Synchronises the
 * stream.  Errors: RTG_ERR_INVALID_ARGUMENT (bad parameters), RTG_ERR_NO_FEASIBLE (nothing
 * collision-free grows from the start: *n_found = 0), RTG_ERR_CUDA.
 */
typedef struct {
    int n_v, n_omega;        /* control grid (3, 5 in the paper)                   */
    float v_max, omega_max;  /* > 0 [m/s], >= 0 [rad/s] (0.6, 0.9)                */
    float dt;                /* primitive duration [s] (1)                         */
    float lambda_t;          /* time weight of the cost (>= 0)                            */
    int samples;             /* collision samples per primitive incl. both ends (>= 2)   */
    int max_depth;           /* primitives per trajectory (>= 1)                          */
    float goal_radius;       /* goal region radius [m] (>= 0)                             */
    float lattice_xy;        /* dedup lattice cell [m] (<= 0: no dedup)                   */
    float lattice_deg;       /* dedup lattice heading cell [deg]                          */
    int beam;                /* frontier nodes kept per layer (>= 1)                      */
    int n_traj;              /* candidates returned (>= 1)                                */
    float z;                 /* height of the robot (and camera) [m]                      */
} rtg_tree_params;
rtg_status rtg_plan_tree(rtg_map map, const float start[3], const float goal[2], const rtg_tree_params* params,
                         void* stream, rtg_traj* out, double* cost, int* n_found, int* reached, long long* stats);

/*
 * Profiling (process-wide).  When enabled, every library phase is bracketed by CUDA events
 * recorded on the stream it is launched on; rtg_profile_read synchronises those events and
 * returns the accumulated device milliseconds and call counts per phase:
 *   0 map build (rtg_map_create), 1 classification, 2 collision (a4), 3 info list,
 *   4 visibility + gain (a5), 5 trajectory reduction (a6), 6 argmax (a7), 7 other.
 * `launches` counts every kernel the library launched since the last reset (profiling on or off).
 */
typedef struct {
    double ms[8];
    long long calls[8];
    long long launches;
} rtg_profile_t;
rtg_status rtg_profile_enable(int on);
rtg_status rtg_profile_read(rtg_profile_t* out, int reset);

const char* rtg_status_string(rtg_status status);
const char* rtg_last_error(void);
/* Library version string, e.g. "rtg 0.1 sm_100a". */
const char* rtg_version(void);

#ifdef __cplusplus
}
#endif
#endif /* RTG_H */
