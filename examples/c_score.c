/* c_score.c -- the boundary used from plain C (no Python, no torch): one planning cycle through
 * include/rtg.h.  A seeded random map of N Gaussians and K straight-ish unicycle trajectories are
 * built on the host, handed to rtg_map_create / rtg_traj_upload as HOST arrays, scored with
 * rtg_score into device buffers the caller owns (cudaMalloc), and reduced with rtg_best.
 *
 * build: gcc -O2 -std=c11 -I include -I /usr/local/cuda/include examples/c_score.c \
 *            -L paper_2409_18122_b200 -lrtg -L /usr/local/cuda/lib64 -lcudart \
 *            -Wl,-rpath,'$ORIGIN/../paper_2409_18122_b200' -lm -o build/c_score
 * run:   build/c_score [N] [K] [T]      (prints "best <index> <score> feasible <count>") */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime_api.h>

#include "rtg.h"

static unsigned long long rng_state = 0x9e3779b97f4a7c15ull;
static double urand(void) {   /* splitmix64 -> [0, 1) */
    unsigned long long z = (rng_state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z ^= z >> 31;
    return (double)(z >> 11) * (1.0 / 9007199254740992.0);
}

#define CK(call)                                                                              \
    do {                                                                                      \
        rtg_status s_ = (call);                                                               \
        if (s_ != RTG_OK && s_ != RTG_ERR_NO_FEASIBLE) {                                      \
            fprintf(stderr, "%s: %s (%s)\n", #call, rtg_status_string(s_), rtg_last_error()); \
            return 1;                                                                         \
        }                                                                                     \
    } while (0)

int main(int argc, char** argv) {
    const long long N = argc > 1 ? atoll(argv[1]) : 100000;
    const int K = argc > 2 ? atoi(argv[2]) : 1024, T = argc > 3 ? atoi(argv[3]) : 50;
    /* map: Gaussians in a 40 x 40 x 3 m box, random orientations and scales, weights U[0,1] */
    float* means = malloc(sizeof(float) * 3 * N);
    float* quats = malloc(sizeof(float) * 4 * N);
    float* scales = malloc(sizeof(float) * 3 * N);
    float* opac = malloc(sizeof(float) * N);
    float* w = malloc(sizeof(float) * N);
    for (long long i = 0; i < N; ++i) {
        means[i] = (float)(40.0 * urand() - 20.0);
        means[N + i] = (float)(40.0 * urand() - 20.0);
        means[2 * N + i] = (float)(3.0 * urand());
        double q[4], qn = 0.0;
        for (int c = 0; c < 4; ++c) { q[c] = urand() - 0.5; qn += q[c] * q[c]; }
        for (int c = 0; c < 4; ++c) quats[c * N + i] = (float)(q[c] / sqrt(qn));
        for (int c = 0; c < 3; ++c) scales[c * N + i] = (float)(0.02 + 0.2 * urand());
        opac[i] = (float)urand();
        w[i] = (float)urand();
    }
    /* trajectories: from the origin at z = 1.5, heading spread over a half-turn, constant speed */
    float* x = malloc(sizeof(float) * K * T);
    float* y = malloc(sizeof(float) * K * T);
    float* z = malloc(sizeof(float) * K * T);
    float* yaw = malloc(sizeof(float) * K * T);
    for (int k = 0; k < K; ++k) {
        const double h = -1.57 + 3.14 * (k + 0.5) / K, v = 0.5 + urand();
        for (int t = 0; t < T; ++t) {
            const double s = v * 0.1 * (t + 1);
            x[k * T + t] = (float)(s * cos(h));
            y[k * T + t] = (float)(s * sin(h));
            z[k * T + t] = 1.5f;
            yaw[k * T + t] = (float)h;
        }
    }
    rtg_robot robot = {0.3f, 3.0f, RTG_COLLIDE_ELLIPSOID};
    rtg_camera cam = {320, 240, 250.f, 250.f, 160.f, 120.f, 0.1f, 6.f};
    rtg_score_params p;
    p.lambda_xi = 1.f; p.k_sigma = 0.5f; p.variant = RTG_VARIANT_XI; p.info_stride = 1;
    p.mode = RTG_MODE_CULLED; p.flags = 0u; p.tau_hi = NAN; p.tau_lo = NAN;
    rtg_map map = NULL;
    rtg_traj traj = NULL;
    CK(rtg_map_create(0, N, RTG_MEM_HOST, means, quats, scales, opac, w, NULL, &robot, NULL, &map));
    CK(rtg_traj_upload(0, K, T, RTG_MEM_HOST, x, y, z, yaw, NULL, &traj));
    int* first_col = NULL;
    unsigned char* feasible = NULL;
    double *gain = NULL, *utility = NULL;
    if (cudaMalloc((void**)&first_col, sizeof(int) * K) || cudaMalloc((void**)&feasible, K) ||
        cudaMalloc((void**)&gain, sizeof(double) * K) || cudaMalloc((void**)&utility, sizeof(double) * K)) {
        fprintf(stderr, "cudaMalloc failed\n");
        return 1;
    }
    CK(rtg_score(map, traj, &cam, &p, first_col, feasible, gain, utility, NULL));
    rtg_best_result best;
    CK(rtg_best(utility, K, 0, NULL, &best));
    unsigned char* hf = malloc(K);
    cudaMemcpy(hf, feasible, K, cudaMemcpyDeviceToHost);
    int nf = 0;
    for (int k = 0; k < K; ++k) nf += hf[k];
    printf("best %lld %.1f feasible %d\n", best.index, best.score, nf);
    rtg_traj_destroy(traj);
    rtg_map_destroy(map);
    cudaFree(first_col); cudaFree(feasible); cudaFree(gain); cudaFree(utility);
    free(means); free(quats); free(scales); free(opac); free(w); free(x); free(y); free(z); free(yaw); free(hf);
    return 0;
}
