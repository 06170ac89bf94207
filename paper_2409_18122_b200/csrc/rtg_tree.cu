// rtg_tree.cu -- on-device motion-primitive tree (§IV-B2).
//
// Trajectory candidates are grown as a tree of unicycle motion primitives (fixed controls over dt,
// N_v x N_omega controls from [0, v_max] x [-omega_max, omega_max]), layer by layer:
// every frontier node is expanded by every control at once and ALL new collision samples of the
// layer are checked against the Gaussian map in one launch ("testing collisions of all sampled
// points with all Gaussians from the map at once while growing the search tree") -- one warp
// per primitive, the exact culled collision test of a4 per sample, stopping at the first collision.
// Between layers the host (C++) keeps the search bookkeeping: cost g = sum (lambda_t + v^2 + w^2) dt
// (Eq. low_level_planner with piecewise-constant u), the minimum-time heuristic
// h = ||p_goal - p|| / v_max, a closed (x, y, heading) lattice keeping the lowest g, a
// beam of the lowest f = g + h nodes, and the goal region ||p - p_goal|| <= goal_radius.  Goal-
// reaching nodes are candidates (not expanded further); the N_traj cheapest are returned,
// or, when none reaches the goal, the N_traj leaves closest to it.  All tie-breaks
// use creation order, so the result is deterministic.
#include <algorithm>
#include <cmath>
#include <unordered_map>
#include <vector>

#include "rtg_host.hpp"

namespace rtg {
namespace {

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

struct ExpandK {
    int M, P, S;        // frontier nodes, controls, samples per primitive (incl. both endpoints)
    double dt;
    float z;
};

// one warp per (node m, control p): samples j = 1 .. S-1 at t_j = j dt / (S-1) (j = 0 is the
// parent's state, checked when it was created); ok = no sample collides; child = state at dt
__global__ void __launch_bounds__(256) k_expand(ExpandK k, const double* __restrict__ fr, const double* __restrict__ ctl,
                                                const CRec* __restrict__ crec, const CMat* __restrict__ cmat,
                                                const CSrc* __restrict__ csrc, const rtg_robot rb,
                                                const int* __restrict__ cstart, ColGridK g, float gq, int n_col,
                                                unsigned char* __restrict__ ok, double* __restrict__ child,
                                                unsigned long long* __restrict__ stats) {
    const int lane = threadIdx.x & 31;
    const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    if (w >= (long long)k.M * k.P) return;
    const int m = (int)(w / k.P), p = (int)(w - (long long)m * k.P);
    const double x0 = fr[4 * m], y0 = fr[4 * m + 1], th0 = fr[4 * m + 2];
    const double v = ctl[2 * p], om = ctl[2 * p + 1];
    unsigned nref = 0;
    unsigned long long ntest = 0;
    bool hit = false;
    int checked = 0;
    double x = x0, y = y0, th = th0;
    for (int j = 1; j < k.S; ++j) {
        const double t = __ddiv_rn(__dmul_rn((double)j, k.dt), (double)(k.S - 1));
        unicycle_at(x0, y0, th0, v, om, t, x, y, th);
        if (!hit && n_col > 0) {
            hit = warp_point_collides(__double2float_rn(x), __double2float_rn(y), k.z, crec, cmat, csrc, rb, cstart,
                                      g, gq, nref, ntest);
            ++checked;
        }
    }
    if (lane == 0) {
        ok[w] = hit ? 0 : 1;
        child[3 * w] = x;
        child[3 * w + 1] = y;
        child[3 * w + 2] = wrap_pi(th);
        if (stats) {
            atomicAdd(&stats[0], (unsigned long long)checked);
            atomicAdd(&stats[1], ntest);
            if (nref) atomicAdd(&stats[2], (unsigned long long)nref);
        }
    }
}

struct Node {
    double x, y, th, g;
    int parent, depth;
};

struct LatticeKey {
    long long a, b, c;
    bool operator==(const LatticeKey& o) const { return a == o.a && b == o.b && c == o.c; }
};
struct LatticeHash {
    size_t operator()(const LatticeKey& k) const {
        return (size_t)(k.a * 73856093LL) ^ (size_t)(k.b * 19349663LL) ^ (size_t)(k.c * 83492791LL);
    }
};

}  // namespace

rtg_status plan_tree(rtg_map_s* m, const float start[3], const float goal[2], const rtg_tree_params& P,
                     cudaStream_t st, std::vector<float>* wx, std::vector<float>* wy, std::vector<float>* wyaw,
                     std::vector<double>* cost, int* reached, long long stats_out[4]) {
    // ---- controls: v on a uniform grid of [0, v_max] incl. endpoints, w likewise on
    // [-w_max, w_max]; a grid of one point is {v_max} / {0}
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
    std::vector<double> pcost(NP);
    for (int p = 0; p < NP; ++p)
        pcost[p] = ((double)P.lambda_t + ctl[2 * p] * ctl[2 * p] + ctl[2 * p + 1] * ctl[2 * p + 1]) * (double)P.dt;
    const double gx = goal[0], gy = goal[1], r2 = (double)P.goal_radius * (double)P.goal_radius;
    auto h_of = [&](double x, double y) { return std::sqrt((gx - x) * (gx - x) + (gy - y) * (gy - y)) / (double)P.v_max; };
    auto at_goal = [&](double x, double y) { return (x - gx) * (x - gx) + (y - gy) * (y - gy) <= r2; };
    const bool dedup = P.lattice_xy > 0 && P.lattice_deg > 0;
    auto key_of = [&](const Node& n) {
        return LatticeKey{(long long)std::floor(n.x / (double)P.lattice_xy), (long long)std::floor(n.y / (double)P.lattice_xy),
                          (long long)std::floor(n.th * (180.0 / M_PI) / (double)P.lattice_deg)};
    };
    std::vector<Node> nodes;
    double th0 = std::remainder((double)start[2], 2.0 * M_PI);   // (-pi, pi]
    if (th0 <= -M_PI) th0 += 2.0 * M_PI;
    nodes.push_back(Node{(double)start[0], (double)start[1], th0, 0.0, -1, 0});
    std::unordered_map<LatticeKey, double, LatticeHash> closed;
    if (dedup) closed[key_of(nodes[0])] = 0.0;
    std::vector<int> frontier, cand;
    if (at_goal(nodes[0].x, nodes[0].y)) cand.push_back(0);   // already in the goal region
    else frontier.push_back(0);
    // ---- device scratch
    ColGridK g;
    g.ox = m->cg.ox; g.oy = m->cg.oy; g.oz = m->cg.oz; g.h = m->cg.h;
    g.R = m->rb_max * (1.0f + 2e-5f) + 1e-4f;
    g.nx = m->cg.nx; g.ny = m->cg.ny; g.nz = m->cg.nz;
    const long long maxM = std::max(1, P.beam);
    double *d_fr = nullptr, *d_ctl = nullptr, *d_child = nullptr;
    unsigned char* d_ok = nullptr;
    unsigned long long* d_stats = nullptr;
    cudaError_t e = dev_alloc((void**)&d_fr, sizeof(double) * 4 * maxM, st);
    if (e == cudaSuccess) e = dev_alloc((void**)&d_ctl, sizeof(double) * 2 * NP, st);
    if (e == cudaSuccess) e = dev_alloc((void**)&d_child, sizeof(double) * 3 * maxM * NP, st);
    if (e == cudaSuccess) e = dev_alloc((void**)&d_ok, maxM * NP, st);
    if (e == cudaSuccess) e = dev_alloc((void**)&d_stats, sizeof(unsigned long long) * 4, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_ctl, ctl.data(), sizeof(double) * 2 * NP, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(d_stats, 0, sizeof(unsigned long long) * 4, st);
    long long expanded = 0;
    std::vector<double> hfr, hchild;
    std::vector<unsigned char> hok;
    for (int depth = 1; depth <= P.max_depth && e == cudaSuccess && !frontier.empty(); ++depth) {
        const int M = (int)frontier.size();
        hfr.assign(4 * (size_t)M, 0.0);
        for (int i = 0; i < M; ++i) {
            const Node& n = nodes[frontier[i]];
            hfr[4 * i] = n.x; hfr[4 * i + 1] = n.y; hfr[4 * i + 2] = n.th; hfr[4 * i + 3] = n.g;
        }
        e = cudaMemcpyAsync(d_fr, hfr.data(), sizeof(double) * 4 * M, cudaMemcpyHostToDevice, st);
        if (e != cudaSuccess) break;
        ExpandK k{M, NP, P.samples, (double)P.dt, P.z};
        const long long warps = (long long)M * NP;
        note_launch(), k_expand<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(
            k, d_fr, d_ctl, m->crec, m->cmat, m->csrc, m->robot, m->cstart, g, m->gq, (int)m->n_col, d_ok, d_child,
            d_stats);
        e = cudaGetLastError();
        if (e != cudaSuccess) break;
        hok.resize(warps);
        hchild.resize(3 * warps);
        e = cudaMemcpyAsync(hok.data(), d_ok, warps, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaMemcpyAsync(hchild.data(), d_child, sizeof(double) * 3 * warps, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) break;
        expanded += M;
        std::vector<int> next;
        for (long long w = 0; w < warps; ++w) {   // creation order: node m ascending, control p ascending
            if (!hok[w]) continue;
            const int mi = (int)(w / NP), p = (int)(w % NP);
            const Node& par = nodes[frontier[mi]];
            Node c{hchild[3 * w], hchild[3 * w + 1], hchild[3 * w + 2], par.g + pcost[p], frontier[mi], depth};
            if (dedup) {
                const LatticeKey key = key_of(c);
                auto it = closed.find(key);
                if (it != closed.end() && it->second <= c.g) continue;
                closed[key] = c.g;
            }
            nodes.push_back(c);
            const int id = (int)nodes.size() - 1;
            if (at_goal(c.x, c.y)) cand.push_back(id);
            else next.push_back(id);
        }
        // beam: lowest f = g + h, ties -> creation order
        std::vector<std::pair<double, int>> fv;
        fv.reserve(next.size());
        for (int id : next) fv.emplace_back(nodes[id].g + h_of(nodes[id].x, nodes[id].y), id);
        std::stable_sort(fv.begin(), fv.end(), [](const std::pair<double, int>& a, const std::pair<double, int>& b) {
            return a.first < b.first;
        });
        if ((long long)fv.size() > maxM) fv.resize(maxM);
        frontier.clear();
        for (auto& pr : fv) frontier.push_back(pr.second);
        std::sort(frontier.begin(), frontier.end());   // keep creation order within the layer
    }
    unsigned long long hs[4] = {0, 0, 0, 0};
    if (e == cudaSuccess) e = cudaMemcpyAsync(hs, d_stats, sizeof(hs), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    dev_free(d_fr, st);
    dev_free(d_ctl, st);
    dev_free(d_child, st);
    dev_free(d_ok, st);
    dev_free(d_stats, st);
    if (e != cudaSuccess) {
        set_error("rtg_plan_tree: %s", cudaGetErrorString(e));
        return e == cudaErrorMemoryAllocation ? RTG_ERR_OUT_OF_MEMORY : RTG_ERR_CUDA;
    }
    // ---- candidates: cheapest goal-reaching nodes, else the leaves closest to the goal
    std::vector<int> pick;
    if (!cand.empty()) {
        *reached = 1;
        pick = cand;
        std::stable_sort(pick.begin(), pick.end(), [&](int a, int b) { return nodes[a].g < nodes[b].g; });
    } else {
        *reached = 0;
        for (int id = 1; id < (int)nodes.size(); ++id) pick.push_back(id);   // every node but the root
        std::stable_sort(pick.begin(), pick.end(), [&](int a, int b) {
            const double ha = h_of(nodes[a].x, nodes[a].y), hb = h_of(nodes[b].x, nodes[b].y);
            if (ha != hb) return ha < hb;
            return nodes[a].g < nodes[b].g;
        });
    }
    if ((int)pick.size() > P.n_traj) pick.resize(P.n_traj);
    const int T = P.max_depth + 1;
    const float nanf_ = std::nanf("");
    wx->assign((size_t)pick.size() * T, nanf_);
    wy->assign((size_t)pick.size() * T, nanf_);
    wyaw->assign((size_t)pick.size() * T, nanf_);
    cost->assign(pick.size(), 0.0);
    for (size_t c = 0; c < pick.size(); ++c) {
        (*cost)[c] = nodes[pick[c]].g;
        for (int id = pick[c]; id >= 0; id = nodes[id].parent) {
            const Node& n = nodes[id];
            (*wx)[c * T + n.depth] = (float)n.x;
            (*wy)[c * T + n.depth] = (float)n.y;
            (*wyaw)[c * T + n.depth] = (float)n.th;
        }
    }
    if (stats_out) {
        stats_out[0] = expanded;
        stats_out[1] = (long long)nodes.size() - 1;
        stats_out[2] = (long long)hs[0];
        stats_out[3] = (long long)hs[1];
    }
    return RTG_OK;
}

}  // namespace rtg
