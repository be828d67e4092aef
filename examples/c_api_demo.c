/* Minimal C client of the C ABI (include/hm.h), no Python: a closed unit cube whose faces are
 * m x m grids of square facets (n = 6 m^2, normals into the cube), one F apply, one solve and one
 * flux evaluation on the GPU, checked against properties that hold exactly or nearly:
 *   - F x on sampled rows equals the direct sum of the one-point entries (eq:Fdef_new_location,
 *     PAPER.md:149-154; on the cube every row sum exceeds 1, so eqn:F_closed leaves F unscaled)
 *     within 10 eps_ACA;
 *   - eps == 1 (black body) gives C = I, so C^-1 b == b;
 *   - a uniform temperature gives q == 0 (Rbar 1 = 0, eq:Rbardef).
 * Build: gcc -O2 -I include examples/c_api_demo.c -L paper_2305_06891_b200 -lhm
 *        -Wl,-rpath,$PWD/paper_2305_06891_b200 -lm -o c_api_demo      (tests/test_gpu_c_api.py) */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "hm.h"

#define CHECK(call)                                                                          \
    do {                                                                                     \
        hm_status st_ = (call);                                                              \
        if (st_ != HM_OK) {                                                                  \
            fprintf(stderr, "%s failed: %s (%s)\n", #call, hm_status_string(st_), hm_last_error(ctx)); \
            return 1;                                                                        \
        }                                                                                    \
    } while (0)

int main(int argc, char** argv) {
    const int m = argc > 1 ? atoi(argv[1]) : 12;
    const int64_t n = 6 * (int64_t)m * m;
    double* xyz = malloc(sizeof(double) * 3 * n);
    double* nrm = malloc(sizeof(double) * 3 * n);
    double* area = malloc(sizeof(double) * n);
    double* box = malloc(sizeof(double) * 6 * n);
    const double h = 1.0 / m;
    int64_t f = 0;
    for (int axis = 0; axis < 3; ++axis)
        for (int side = 0; side < 2; ++side)
            for (int a = 0; a < m; ++a)
                for (int b = 0; b < m; ++b, ++f) {
                    const int u = (axis + 1) % 3, v = (axis + 2) % 3;
                    double c[3];
                    c[axis] = side;
                    c[u] = (a + 0.5) * h;
                    c[v] = (b + 0.5) * h;
                    for (int d = 0; d < 3; ++d) {
                        xyz[3 * f + d] = c[d];
                        nrm[3 * f + d] = d == axis ? (side ? -1.0 : 1.0) : 0.0;
                        box[6 * f + d] = c[d] - (d == axis ? 0.0 : 0.5 * h);
                        box[6 * f + 3 + d] = c[d] + (d == axis ? 0.0 : 0.5 * h);
                    }
                    area[f] = h * h;
                }
    hm_ctx* ctx = NULL;
    hm_status s0 = hm_init(0, 0, 1, NULL, 0, &ctx);
    if (s0 != HM_OK) {
        fprintf(stderr, "hm_init: %s\n", hm_status_string(s0));
        return 1;
    }
    hm_tree_params tp = {64, 1.0, 0};
    hm_geom* g = NULL;
    CHECK(hm_build_geometry(ctx, n, xyz, nrm, area, box, &tp, &g));
    hm_aca_params ap = {1e-6, 0, 1, 0, 0, 0};
    hm_hmat* F = NULL;
    CHECK(hm_assemble_aca(ctx, g, &ap, &F));
    double* one = malloc(sizeof(double) * n);
    double* y = malloc(sizeof(double) * n);
    double* eps = malloc(sizeof(double) * n);
    for (int64_t i = 0; i < n; ++i) { one[i] = 1.0; eps[i] = 1.0; }
    for (int64_t i = 0; i < n; ++i) one[i] = 1.0 + 0.5 * sin(0.37 * i);
    CHECK(hm_apply_F(ctx, F, 1, one, y, NULL));
    double e2 = 0.0, r2 = 0.0;
    for (int64_t i = 0; i < n; i += 7) {   // direct one-point sums on sampled rows
        double acc = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            if (j == i) continue;
            const double dx = xyz[3 * j] - xyz[3 * i], dy = xyz[3 * j + 1] - xyz[3 * i + 1], dz = xyz[3 * j + 2] - xyz[3 * i + 2];
            const double rr = dx * dx + dy * dy + dz * dz;
            const double ci = nrm[3 * i] * dx + nrm[3 * i + 1] * dy + nrm[3 * i + 2] * dz;
            const double cj = -(nrm[3 * j] * dx + nrm[3 * j + 1] * dy + nrm[3 * j + 2] * dz);
            if (ci > 0.0 && cj > 0.0) acc += area[i] * area[j] * ci * cj / (M_PI * rr * rr) * one[j];
        }
        e2 += (y[i] - acc) * (y[i] - acc);
        r2 += acc * acc;
    }
    const double dev = sqrt(e2 / r2);
    hm_lu_params lp = {1e-6, -1};
    hm_hlu* LU = NULL;
    CHECK(hm_factor_hlu(ctx, F, eps, &lp, &LU));
    double* z = malloc(sizeof(double) * n);
    for (int64_t i = 0; i < n; ++i) y[i] = sin(0.1 * i);
    CHECK(hm_solve_C(ctx, LU, 1, y, z, NULL));
    double dz = 0.0;
    for (int64_t i = 0; i < n; ++i) dz = fmax(dz, fabs(z[i] - y[i]));
    double* T = malloc(sizeof(double) * n);
    for (int64_t i = 0; i < n; ++i) T[i] = 600.0;
    CHECK(hm_radiative_flux(ctx, F, LU, 1, T, z, NULL));
    double dq = 0.0;
    for (int64_t i = 0; i < n; ++i) dq = fmax(dq, fabs(z[i]));
    hm_storage st;
    CHECK(hm_storage_report(F, LU, &st));
    printf("n %lld blocks %lld lowrank %lld bytes_F %lld | F x vs direct sums (sampled rows) %.3e | black body max |z - b| %.3e | "
           "uniform T max |q| %.3e W/m^2 (sigma T^4 = %.1f)\n",
           (long long)n, (long long)st.n_blocks, (long long)st.n_lowrank, (long long)st.bytes_F, dev, dz, dq,
           5.670374419e-8 * pow(600.0, 4));
    hm_destroy_hlu(LU);
    hm_destroy_hmat(F);
    hm_destroy_geom(g);
    hm_finalize(ctx);
    const int ok = dev < 1e-5 && dz < 1e-12 && dq < 1e-9 * 5.670374419e-8 * pow(600.0, 4);
    printf("%s\n", ok ? "OK" : "FAIL");
    return ok ? 0 : 1;
}
