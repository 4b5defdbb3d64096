/*
 * c_abi_demo.c — the B200 sweep driven from plain C through the C ABI
 * (include/stencil_b200.h), no Python and no torch: the boundary a native
 * host (or the reference's ctypes binding) sees.
 *
 *   gcc -O2 -ffp-contract=off -I include examples/c_abi_demo.c \
 *       -L paper_1308_1343_b200 -lstencil_b200 -L /usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_1308_1343_b200:/usr/local/cuda/lib64 -o c_abi_demo
 *   ./c_abi_demo
 *
 * It sweeps (1) the reference's 7-point kernel (_update_rows,
 * stencil.py:31-39) over a 64^3 box and (2) the 4th-order ten-output set
 * over a 40x24x16 box, copies the results back with the library's own
 * host<->device copies, and compares them byte for byte with the same
 * expression trees evaluated here on the CPU (one IEEE rounding per
 * operation, the reference's association, no FMA contraction).
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "stencil_b200.h"

#define CHECK(call)                                                                    \
    do {                                                                               \
        int rc_ = (call);                                                              \
        if (rc_ != SB_OK) {                                                            \
            fprintf(stderr, "%s failed (%d): %s\n", #call, rc_, sb_last_error());      \
            exit(1);                                                                   \
        }                                                                              \
    } while (0)

/* A device grid in the library's layout: xpad = 16 readable elements before
 * x = 0 (rows start 128-byte aligned), row pitch a multiple of 16. */
static sb_array make_grid(int nx, int ny, int nz, int ghost, double **base) {
    sb_array a;
    const int64_t xpad = 16;
    a.sy = ((xpad + nx + ghost) + 15) / 16 * 16;
    a.sz = a.sy * (ny + 2 * ghost);
    a.nx = nx;
    a.ny = ny;
    a.nz = nz;
    a.ghost = ghost;
    a.xpad = (int32_t)xpad;
    const size_t n = (size_t)a.sz * (size_t)(nz + 2 * ghost);
    if (cudaMalloc((void **)base, n * sizeof(double)) != cudaSuccess) {
        fprintf(stderr, "cudaMalloc failed\n");
        exit(1);
    }
    a.origin = *base + xpad + (int64_t)ghost * a.sy + (int64_t)ghost * a.sz;
    return a;
}

/* deterministic values in [-1, 1) */
static double next_value(uint64_t *s) {
    *s = *s * 6364136223846793005ULL + 1442695040888963407ULL;
    return (double)(*s >> 11) * (2.0 / 9007199254740992.0) - 1.0;
}

/* dense (z,y,x) host field of (n+2g)^3 points including ghosts */
static double *host_field(int nx, int ny, int nz, int g, uint64_t seed) {
    const size_t n = (size_t)(nx + 2 * g) * (ny + 2 * g) * (nz + 2 * g);
    double *h = (double *)malloc(n * sizeof(double));
    for (size_t i = 0; i < n; ++i) h[i] = next_value(&seed);
    return h;
}

#define AT(h, x, y, z, W, H) (h)[(size_t)(z) * (H) * (W) + (size_t)(y) * (W) + (x)]

int main(void) {
    CHECK(sb_init(0));
    if (sb_abi_version() != SB_ABI_VERSION) {
        fprintf(stderr, "library ABI %d, header %d\n", sb_abi_version(), SB_ABI_VERSION);
        return 1;
    }
    int failures = 0;

    /* ---- (1) 7-point Laplacian, 64^3, h = 1/64: C0 = -6/h^2, C1 = 1/h^2 ---- */
    {
        const int n = 64, g = 1, W = n + 2;
        const double c0 = -6.0 * 64.0 * 64.0, c1 = 64.0 * 64.0;
        double *bs, *bd;
        sb_array src = make_grid(n, n, n, g, &bs), dst = make_grid(n, n, n, g, &bd);
        double *h = host_field(n, n, n, g, 20130715);
        CHECK(sb_copy_h2d(src, h, 1, NULL));
        sb_space sp = {{0, 0, 0}, {n, n, n}};
        sb_launch p = {64, 8, 2, 0};
        CHECK(sb_lap7(dst, src, sp, c0, c1, p, NULL));
        double *got = (double *)malloc((size_t)n * n * n * sizeof(double));
        CHECK(sb_copy_d2h(got, dst, 0, NULL));
        if (cudaDeviceSynchronize() != cudaSuccess) return 1;
        size_t bad = 0;
        for (int z = 0; z < n; ++z)
            for (int y = 0; y < n; ++y)
                for (int x = 0; x < n; ++x) {
                    const int X = x + g, Y = y + g, Z = z + g;
                    /* stencil.py:35-39: C0*b + C1*(((xm+xp)+(ym+yp))+(zm+zp)) */
                    const double b = AT(h, X, Y, Z, W, W);
                    const double sx = AT(h, X - 1, Y, Z, W, W) + AT(h, X + 1, Y, Z, W, W);
                    const double sy = AT(h, X, Y - 1, Z, W, W) + AT(h, X, Y + 1, Z, W, W);
                    const double sz = AT(h, X, Y, Z - 1, W, W) + AT(h, X, Y, Z + 1, W, W);
                    const double want = c0 * b + c1 * ((sx + sy) + sz);
                    const double v = got[((size_t)z * n + y) * n + x];
                    bad += memcmp(&v, &want, sizeof v) != 0;
                }
        printf("lap7 64^3: %s (%zu of %d points differ)\n", bad ? "MISMATCH" : "bit-identical", bad, n * n * n);
        failures += bad != 0;
        free(got);
        free(h);
        cudaFree(bs);
        cudaFree(bd);
    }

    /* ---- (2) 4th-order ten-output set, 40 x 24 x 16, h = 1/40: Lap4 and Dxy checked ---- */
    {
        const int nx = 40, ny = 24, nz = 16, g = 2, W = nx + 4, H = ny + 4;
        const double hh = 1.0 / 40.0;
        sb_d4_constants k = {1.0 / (12.0 * hh), 1.0 / (12.0 * hh * hh), 1.0 / (144.0 * hh * hh)};
        double *bs, *bo[SB_N_D4_OUT];
        sb_array src = make_grid(nx, ny, nz, g, &bs), out[SB_N_D4_OUT];
        for (int i = 0; i < SB_N_D4_OUT; ++i) out[i] = make_grid(nx, ny, nz, 0, &bo[i]);
        double *h = host_field(nx, ny, nz, g, 7);
        CHECK(sb_copy_h2d(src, h, 1, NULL));
        sb_space sp = {{0, 0, 0}, {nx, ny, nz}};
        sb_launch p = {32, 4, 4, 0};
        CHECK(sb_d4_all(out, src, sp, k, p, NULL));
        const size_t npts = (size_t)nx * ny * nz;
        double *lap = (double *)malloc(npts * sizeof(double)), *dxy = (double *)malloc(npts * sizeof(double));
        CHECK(sb_copy_d2h(lap, out[9], 0, NULL));
        CHECK(sb_copy_d2h(dxy, out[6], 0, NULL));
        if (cudaDeviceSynchronize() != cudaSuccess) return 1;
        size_t bad = 0;
#define U(dx, dy, dz) AT(h, X + (dx), Y + (dy), Z + (dz), W, H)
        for (int z = 0; z < nz; ++z)
            for (int y = 0; y < ny; ++y)
                for (int x = 0; x < nx; ++x) {
                    const int X = x + g, Y = y + g, Z = z + g;
                    /* D2 = ((16(u[-1]+u[+1]) - (u[-2]+u[+2])) - 30u) k2, Lap4 = (Dxx+Dyy)+Dzz */
                    const double c30 = 30.0 * U(0, 0, 0);
                    const double dxx = ((16.0 * (U(-1, 0, 0) + U(1, 0, 0)) - (U(-2, 0, 0) + U(2, 0, 0))) - c30) * k.k2;
                    const double dyy = ((16.0 * (U(0, -1, 0) + U(0, 1, 0)) - (U(0, -2, 0) + U(0, 2, 0))) - c30) * k.k2;
                    const double dzz = ((16.0 * (U(0, 0, -1) + U(0, 0, 1)) - (U(0, 0, -2) + U(0, 0, 2))) - c30) * k.k2;
                    const double want_lap = (dxx + dyy) + dzz;
                    /* D_xy = d1u_y(d1u_x) k11, d1u = (u[-2]-u[+2]) + 8(u[+1]-u[-1]) along x first */
                    double r[5];
                    for (int j = -2; j <= 2; ++j)
                        r[j + 2] = (U(-2, j, 0) - U(2, j, 0)) + 8.0 * (U(1, j, 0) - U(-1, j, 0));
                    const double want_dxy = ((r[0] - r[4]) + 8.0 * (r[3] - r[1])) * k.k11;
                    const size_t i = ((size_t)z * ny + y) * nx + x;
                    bad += memcmp(&lap[i], &want_lap, 8) != 0;
                    bad += memcmp(&dxy[i], &want_dxy, 8) != 0;
                }
#undef U
        printf("d4_all 40x24x16 (Lap4, Dxy): %s (%zu of %zu values differ)\n", bad ? "MISMATCH" : "bit-identical", bad,
               2 * npts);
        failures += bad != 0;
        free(lap);
        free(dxy);
        free(h);
        cudaFree(bs);
        for (int i = 0; i < SB_N_D4_OUT; ++i) cudaFree(bo[i]);
    }
    CHECK(sb_shutdown());
    return failures ? 1 : 0;
}
