/*
 * A plain C client of the C ABI (include/nlse.h): create a 3D 2SHOC MSD context, upload a
 * field read from a file, step it with the recommended k, read it back and write it out, and
 * print k, mass and Hamiltonian.  Built by tests/test_abi.py (gcc: the header compiles as C and
 * every call links) and run by the GPU test, which compares the field with the oracle bit for bit.
 *
 *   abi_demo <nx> <ny> <nz> <nsteps> <in.bin> <out.bin>     (complex128, x fastest)
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "nlse.h"

static int check(nlse_status st, const nlse_ctx *ctx, const char *what)
{
    if (st != NLSE_OK) {
        fprintf(stderr, "%s: %s: %s\n", what, nlse_status_string(st), nlse_last_error(ctx));
        return 1;
    }
    return 0;
}

int main(int argc, char **argv)
{
    if (argc != 7) { fprintf(stderr, "usage: abi_demo nx ny nz nsteps in.bin out.bin\n"); return 2; }
    const int64_t dims[3] = {atol(argv[1]), atol(argv[2]), atol(argv[3])};
    const int64_t nsteps = atol(argv[4]);
    const int64_t n = dims[0] * dims[1] * dims[2];
    const double h = 0.5, a = 1.0, s = -1.0;
    double kmax = 0, krec = 0;
    if (check(nlse_stability_bound(3, a, h, NLSE_2SHOC4, &kmax, &krec), NULL, "nlse_stability_bound")) return 1;
    double *psi = malloc(sizeof(double) * 2 * (size_t)n);
    FILE *fi = fopen(argv[5], "rb");
    if (!psi || !fi || fread(psi, sizeof(double), 2 * (size_t)n, fi) != 2 * (size_t)n) return 1;
    fclose(fi);
    nlse_ctx *ctx = NULL;
    if (check(nlse_create(3, dims, h, a, s, NULL, NLSE_BC_MSD, NLSE_2SHOC4, NLSE_FP64, 0, &ctx), NULL, "nlse_create"))
        return 1;
    int rc = check(nlse_set_psi(ctx, psi), ctx, "nlse_set_psi") ||
             check(nlse_step(ctx, krec, nsteps), ctx, "nlse_step") ||
             check(nlse_get_psi(ctx, psi), ctx, "nlse_get_psi");
    double mass = 0, ham = 0;
    if (!rc) rc = check(nlse_diagnostics(ctx, &mass, &ham), ctx, "nlse_diagnostics");
    nlse_destroy(ctx);
    if (rc) return 1;
    FILE *f = fopen(argv[6], "wb");
    if (!f || fwrite(psi, sizeof(double), 2 * (size_t)n, f) != 2 * (size_t)n) return 1;
    fclose(f);
    printf("k %.17g mass %.17g hamiltonian %.17g\n", krec, mass, ham);
    free(psi);
    return 0;
}
