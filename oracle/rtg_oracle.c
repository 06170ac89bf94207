/*
 * rtg_oracle.c -- plain, slow, obviously-correct CPU oracle for RT-GuIDE's
 * trajectory-scoring hot path (arXiv 2409.18122), in double precision.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load or call this code.
 * The product path (paper_2409_18122_b200/, librtg.so) never does; it shares no
 * code, header, table or helper with this file.
 *
 * What it computes (every step cites PAPER.md lines):
 *   O1  per Gaussian: unit quaternion -> rotation R, inflated semi-axes
 *       a_i = lambda_g * s_i + r_robot
 *   O2  per (waypoint p, Gaussian g) collision quadratic form
 *       q = sum_i ((R^T (p - mu))_i / a_i)^2, collide <=> q < 1
 *       (isotropic: ||p-mu|| < r_robot + lambda_g r);
 *       PRINCIPAL_AXIS variant: ||p-mu|| < lambda_g max_i s_i + r_robot
 *   O3  per (waypoint, Gaussian) binary visibility v(x,g): the mean projects
 *       inside the image with depth in [z_near, z_far], no occlusion
 *       (PAPER.md:137-140 projection, 214 binary J, 256-257 range culling)
 *   O4  classification H / L / O at mean +- k_sigma std
 *   O5  per waypoint: collision flags, trace-proxy gain sum_{visible} u_g
 *       (Eq. eq:nbv with binary J) and the counts that give
 *       xi = n_H - lambda_xi n_L (Eq. equ:view_util)
 * The per-trajectory reduction and the argmax (O6, O7; Eq. equ:traj_utility,
 * PAPER.md:312-320) are written out in numpy in oracle/oracle.py.
 *
 * Decisions are taken in double.  Every decision also reports whether it lies
 * inside the north_star ambiguity band (|q-1| <= 1e-6, |sigma_j| <= 1e-6 scale_j),
 * so tests can tell a genuine mismatch from a rounding-level one.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#define ORC_BAND 1e-6

/* O1: Hamilton rotation matrix of the normalised quaternion (w,x,y,z). */
static void orc_rotation(const double q_in[4], double R[3][3]) {
    double n = sqrt(q_in[0] * q_in[0] + q_in[1] * q_in[1] + q_in[2] * q_in[2] + q_in[3] * q_in[3]);
    double w = q_in[0] / n, x = q_in[1] / n, y = q_in[2] / n, z = q_in[3] / n;
    R[0][0] = 1.0 - 2.0 * (y * y + z * z);
    R[0][1] = 2.0 * (x * y - w * z);
    R[0][2] = 2.0 * (x * z + w * y);
    R[1][0] = 2.0 * (x * y + w * z);
    R[1][1] = 1.0 - 2.0 * (x * x + z * z);
    R[1][2] = 2.0 * (y * z - w * x);
    R[2][0] = 2.0 * (x * z - w * y);
    R[2][1] = 2.0 * (y * z + w * x);
    R[2][2] = 1.0 - 2.0 * (x * x + y * y);
}

/* O2: collision quadratic form q for one pair.  rule 0 = inflated ellipsoid,
 * rule 1 = principal axis as radius.  mu/quat/s are one Gaussian's fp32 inputs. */
double orc_collision_q(const double mu[3], const double quat[4], const double s[3],
                       double r_robot, double lambda_g, int rule, const double p[3]) {
    double d[3] = {p[0] - mu[0], p[1] - mu[1], p[2] - mu[2]};
    if (rule == 1) {
        double smax = s[0];
        if (s[1] > smax) smax = s[1];
        if (s[2] > smax) smax = s[2];
        double gamma = lambda_g * smax + r_robot;          /* gamma := r_robot + lambda_g r */
        return (d[0] * d[0] + d[1] * d[1] + d[2] * d[2]) / (gamma * gamma);
    }
    double R[3][3];
    orc_rotation(quat, R);
    double q = 0.0;
    for (int i = 0; i < 3; ++i) {
        double a_i = lambda_g * s[i] + r_robot;            /* inflated semi-axis */
        double e_i = (R[0][i] * d[0] + R[1][i] * d[1] + R[2][i] * d[2]) / a_i;   /* (R^T d)_i / a_i */
        q += e_i * e_i;
    }
    return q;
}

/* O3: the six frustum slacks of one pair.  cam = {W, H, fx, fy, cx, cy, z_near, z_far};
 * pose = {x, y, z, yaw}.  Camera at the waypoint, optical axis (cos yaw, sin yaw, 0),
 * x right = (sin yaw, -cos yaw, 0), y down = (0,0,-1).
 * visible <=> all sigma_j >= 0, i.e. u = fx X/Z + cx in [0,W], v = fy Y/Z + cy in [0,H],
 * z_near <= Z <= z_far (d = e3^T R^T (mu - T)). */
void orc_visibility_slacks(const double mu[3], const double pose[4], const double cam[8],
                           double sigma[6], double scale[6]) {
    double W = cam[0], H = cam[1], fx = cam[2], fy = cam[3], cx = cam[4], cy = cam[5];
    double zn = cam[6], zf = cam[7];
    double c = cos(pose[3]), s = sin(pose[3]);
    double dx = mu[0] - pose[0], dy = mu[1] - pose[1], dz = mu[2] - pose[2];
    double Z = c * dx + s * dy;
    double X = s * dx - c * dy;
    double Y = -dz;
    sigma[0] = Z - zn;
    sigma[1] = zf - Z;
    sigma[2] = fx * X + cx * Z;
    sigma[3] = (W - cx) * Z - fx * X;
    sigma[4] = fy * Y + cy * Z;
    sigma[5] = (H - cy) * Z - fy * Y;
    double aZ = fabs(Z);
    scale[0] = aZ > zn ? aZ : zn;
    scale[1] = aZ > zf ? aZ : zf;
    double mx = cx > (W - cx) ? cx : (W - cx);
    double my = cy > (H - cy) ? cy : (H - cy);
    scale[2] = scale[3] = fx * fabs(X) + mx * aZ;
    scale[4] = scale[5] = fy * fabs(Y) + my * aZ;
}

/* visibility decision: returns nominal (all sigma >= 0); *amb = band case.  A pose with any
 * non-finite coordinate (trajectory padding) sees nothing, definitely: no slack is evaluated, so
 * no infinite slack/scale pair can report a band case (reading R8). */
static int orc_visible(const double mu[3], const double pose[4], const double cam[8], int* amb) {
    double sg[6], sc[6];
    if (!(isfinite(pose[0]) && isfinite(pose[1]) && isfinite(pose[2]) && isfinite(pose[3]))) {
        *amb = 0;
        return 0;
    }
    orc_visibility_slacks(mu, pose, cam, sg, sc);
    int nominal = 1, definitely_out = 0, near = 0;
    for (int j = 0; j < 6; ++j) {
        if (!(sg[j] >= 0.0)) nominal = 0;
        if (sg[j] < -ORC_BAND * sc[j]) definitely_out = 1;
        if (fabs(sg[j]) <= ORC_BAND * sc[j]) near = 1;
    }
    *amb = (!definitely_out) && near;
    return nominal;
}

/* O4: classification into H (+1), L (-1), O (0); ineligible (NO_GAIN) -> 2.
 * u = w (variant 0 XI, 1 SUM) or w^2 (variant 2 SQ).
 * m = mean u, s = population std (two-pass), tau_hi = m + k s, tau_lo = m - k s
 * (PAPER.md:328); a non-NaN tau_in overrides.  Strict inequalities. */
int orc_classify(long long n, const float* info_w, const unsigned char* flags, int variant,
                 double k_sigma, double tau_hi_in, double tau_lo_in, double* tau_out,
                 signed char* cls, unsigned char* cls_amb, double* u_out) {
    long long cnt = 0;
    double sum = 0.0;
    for (long long g = 0; g < n; ++g) {
        double u = (double)info_w[g];
        if (variant == 2) u = u * u;
        u_out[g] = u;
        if (flags && (flags[g] & 2u)) continue;
        sum += u;
        cnt += 1;
    }
    double m = cnt ? sum / (double)cnt : 0.0;
    double ss = 0.0;
    for (long long g = 0; g < n; ++g) {
        if (flags && (flags[g] & 2u)) continue;
        double dlt = u_out[g] - m;
        ss += dlt * dlt;
    }
    double sd = cnt ? sqrt(ss / (double)cnt) : 0.0;
    double th = m + k_sigma * sd, tl = m - k_sigma * sd;
    if (!isnan(tau_hi_in)) th = tau_hi_in;
    if (!isnan(tau_lo_in)) tl = tau_lo_in;
    tau_out[0] = th;
    tau_out[1] = tl;
    tau_out[2] = m;
    tau_out[3] = sd;
    for (long long g = 0; g < n; ++g) {
        if (flags && (flags[g] & 2u)) { cls[g] = 2; cls_amb[g] = 0; continue; }
        double u = u_out[g];
        cls[g] = u > th ? 1 : (u < tl ? -1 : 0);
        cls_amb[g] = (fabs(u - th) <= 1e-12 * fabs(th)) || (fabs(u - tl) <= 1e-12 * fabs(tl));
    }
    return 0;
}

/* O5: every waypoint against every Gaussian.
 * Inputs: the map (planar SoA as in include/rtg.h), cls/u from orc_classify,
 * robot {r_robot, lambda_g}, rule, cam[8], nwp flattened waypoints.
 * do_collision = 0 skips O2 (gain-only viewpoints).
 * Outputs per waypoint (arrays of length nwp):
 *   col[3*i + {0,1,2}] = {nominal collision, definite collision, ambiguous-only}
 *   n_col[i]           = number of nominal colliding Gaussians
 *   gain[3*i + {0,1,2}] = {nominal, lo, hi} sum of u over visible eligible Gaussians
 *   nh[3*i+{..}], nl[3*i+{..}] = {nominal, lo, hi} visible H / L counts
 *   amb[2*i + {0,1}]   = number of ambiguous collision / visibility pairs */
int orc_waypoints(long long n, const float* means, const float* quats, const float* scales,
                  const unsigned char* flags, const signed char* cls, const double* u,
                  double r_robot, double lambda_g, int rule, const double* cam,
                  long long nwp, const float* wx, const float* wy, const float* wz, const float* wyaw,
                  int do_collision,
                  unsigned char* col, int* n_col, double* gain, long long* nh, long long* nl,
                  long long* amb) {
#pragma omp parallel for schedule(dynamic, 4)
    for (long long i = 0; i < nwp; ++i) {
        double p[3] = {wx[i], wy[i], wz[i]};
        double pose[4] = {wx[i], wy[i], wz[i], wyaw[i]};
        int c_nom = 0, c_def = 0, c_amb = 0, cnt = 0;
        double g_nom = 0.0, g_lo = 0.0, g_hi = 0.0;
        long long h_nom = 0, h_lo = 0, h_hi = 0, l_nom = 0, l_lo = 0, l_hi = 0;
        long long a_col = 0, a_vis = 0;
        for (long long g = 0; g < n; ++g) {
            double mu[3] = {means[g], means[n + g], means[2 * n + g]};
            unsigned f = flags ? flags[g] : 0u;
            if (do_collision && !(f & 1u)) {
                double qt[4] = {quats[g], quats[n + g], quats[2 * n + g], quats[3 * n + g]};
                double sc[3] = {scales[g], scales[n + g], scales[2 * n + g]};
                double q = orc_collision_q(mu, qt, sc, r_robot, lambda_g, rule, p);
                int nominal = q < 1.0;
                int in_band = fabs(q - 1.0) <= ORC_BAND;
                c_nom |= nominal;
                cnt += nominal;
                if (nominal && !in_band) c_def = 1;
                if (in_band) { c_amb = 1; a_col += 1; }
            }
            if (!(f & 2u)) {
                int ab;
                int vis = orc_visible(mu, pose, cam, &ab);
                int definite = vis && !ab;
                if (ab) a_vis += 1;
                if (vis) {
                    g_nom += u[g];
                    h_nom += cls[g] == 1;
                    l_nom += cls[g] == -1;
                }
                if (definite) {
                    g_lo += u[g];
                    h_lo += cls[g] == 1;
                    l_lo += cls[g] == -1;
                }
                if (definite || ab) {
                    g_hi += u[g];
                    h_hi += cls[g] == 1;
                    l_hi += cls[g] == -1;
                }
            }
        }
        col[3 * i + 0] = (unsigned char)c_nom;
        col[3 * i + 1] = (unsigned char)c_def;
        col[3 * i + 2] = (unsigned char)(!c_def && c_amb);
        n_col[i] = cnt;
        gain[3 * i + 0] = g_nom; gain[3 * i + 1] = g_lo; gain[3 * i + 2] = g_hi;
        nh[3 * i + 0] = h_nom; nh[3 * i + 1] = h_lo; nh[3 * i + 2] = h_hi;
        nl[3 * i + 0] = l_nom; nl[3 * i + 1] = l_lo; nl[3 * i + 2] = l_hi;
        amb[2 * i + 0] = a_col; amb[2 * i + 1] = a_vis;
    }
    return 0;
}

/* Full pair collision mask (tiny inputs): mask[i*n + g] = nominal collide,
 * band[i*n + g] = |q - 1| <= 1e-6.  NO_COLLIDE Gaussians give 0. */
int orc_pair_mask(long long n, const float* means, const float* quats, const float* scales,
                  const unsigned char* flags, double r_robot, double lambda_g, int rule,
                  long long nwp, const float* wx, const float* wy, const float* wz,
                  unsigned char* mask, unsigned char* band) {
#pragma omp parallel for schedule(static)
    for (long long i = 0; i < nwp; ++i) {
        double p[3] = {wx[i], wy[i], wz[i]};
        for (long long g = 0; g < n; ++g) {
            mask[i * n + g] = 0;
            band[i * n + g] = 0;
            if (flags && (flags[g] & 1u)) continue;
            double mu[3] = {means[g], means[n + g], means[2 * n + g]};
            double qt[4] = {quats[g], quats[n + g], quats[2 * n + g], quats[3 * n + g]};
            double sc[3] = {scales[g], scales[n + g], scales[2 * n + g]};
            double q = orc_collision_q(mu, qt, sc, r_robot, lambda_g, rule, p);
            mask[i * n + g] = q < 1.0;
            band[i * n + g] = fabs(q - 1.0) <= ORC_BAND;
        }
    }
    return 0;
}

/* Unicycle motion primitive, closed form of
 * p' = v (cos th, sin th), th' = omega, sampled at t_l = (l+1) dt.
 * Heading wrapped to (-pi, pi]. */
void orc_unicycle(double x0, double y0, double z0, double th0, double v, double omega,
                  double dt, int T, double* x, double* y, double* z, double* yaw) {
    for (int l = 0; l < T; ++l) {
        double t = (l + 1) * dt;
        double th = th0 + omega * t;
        if (fabs(omega) < 1e-12) {
            x[l] = x0 + v * t * cos(th0);
            y[l] = y0 + v * t * sin(th0);
        } else {
            x[l] = x0 + (v / omega) * (sin(th) - sin(th0));
            y[l] = y0 + (v / omega) * (cos(th0) - cos(th));
        }
        z[l] = z0;
        double w = fmod(th + M_PI, 2.0 * M_PI);
        if (w < 0) w += 2.0 * M_PI;
        w -= M_PI;
        if (w <= -M_PI) w += 2.0 * M_PI;
        yaw[l] = w;
    }
}
