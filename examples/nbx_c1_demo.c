/* A host program in plain C against the drop-in boundary (include/nbx.h + libnbx.so),
 * no Python: the reference's acceptance toy (C1, test_acceptance.py:52-65)
 * rendered on the GPU through nbx_spots, once per compute path, plus a plan re-run.
 *
 *   cc -O2 -I include examples/nbx_c1_demo.c -L paper_2205_07976_b200/_lib -lnbx \
 *      -Wl,-rpath,$PWD/paper_2205_07976_b200/_lib -lm -o nbx_c1_demo
 *   ./nbx_c1_demo out_prefix      # writes out_prefix.fp64.f32 / .fp32.f32 (raw float32 images)
 *
 * The crystal is UnitCell(100, 100, 100, 90, 90, 90) with the identity orientation and one
 * mosaic domain, N = (5, 5, 5), Fhkl {(1,0,0): 250} default 100; the panel is 256^2 at 100 um,
 * 0.1 m, beam centre (127.5, 127.5); one wavelength of 1 A, weight 1, fluence 1e24,
 * polarisation on.  tests/test_gpu_c_api.py compares the images with the Python API's.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "nbx.h"

static int check(void* ctx, int status, int64_t first_bad, const char* what) {
    if (status == NBX_OK) return 0;
    fprintf(stderr, "%s: status %d (%s), first bad pixel %lld\n", what, status, nbx_last_error(ctx),
            (long long)first_bad);
    return 1;
}

int main(int argc, char** argv) {
    const char* prefix = argc > 1 ? argv[1] : "nbx_c1";
    const double deg = 3.14159265358979323846 / 180.0;
    /* real-space rows a, b, c: a along x, b in the x-y plane (model.py:90-110) */
    const double A = 100.0, B = 100.0, C = 100.0;
    const double ca = cos(90.0 * deg), cb = cos(90.0 * deg), cg = cos(90.0 * deg), sg = sin(90.0 * deg);
    const double factor = 1.0 - ca * ca - cb * cb - cg * cg + 2.0 * ca * cb * cg;
    const double bases[9] = {A, 0.0, 0.0, B * cg, B * sg, 0.0, C * cb, C * (ca - cb * cg) / sg, C * sqrt(factor) / sg};

    nbx_panel panel = {0};
    panel.slow_pixels = 256;
    panel.fast_pixels = 256;
    panel.thick_steps = 1;
    panel.pixel_size = 100e-6;
    panel.distance = 0.1;
    panel.beam_center[0] = 127.5;
    panel.beam_center[1] = 127.5;
    panel.fast_axis[0] = 1.0;
    panel.slow_axis[1] = 1.0;

    const double wavelengths[1] = {1.0}, weights[1] = {1.0};
    const int32_t hkl[3] = {1, 0, 0};
    const double amplitudes[1] = {250.0};

    nbx_spots_desc d = {0};
    d.n_panels = 1;
    d.oversample = 1;
    d.panels = &panel;
    d.beam_direction[2] = 1.0;
    d.polarization_on = 1;
    d.n_sources = 1;
    d.wavelengths = wavelengths;
    d.weights = weights;
    d.fluence = 1e24;
    d.r_e_sqr = 7.94079248e-30; /* kernels.py:44 */
    d.n_domains = 1;
    d.shape = NBX_SHAPE_SINCG;
    d.bases = bases;
    d.n_cells[0] = d.n_cells[1] = d.n_cells[2] = 5;
    d.n_entries = 1;
    d.hkl = hkl;
    d.amplitudes = amplitudes;
    d.default_f = 100.0;

    if (nbx_device_count() < 1) {
        fprintf(stderr, "no CUDA device\n");
        return 2;
    }
    void* ctx = nbx_ctx_create(0);
    if (!ctx) {
        fprintf(stderr, "nbx_ctx_create: %s\n", nbx_last_error(NULL));
        return 2;
    }
    const int64_t n = nbx_output_pixels(&d);
    float* img = (float*)malloc((size_t)n * sizeof(float));
    float* again = (float*)malloc((size_t)n * sizeof(float));
    int rc = 0;
    const char* names[2] = {"fp64", "fp32"};
    for (int compute = 0; compute < 2 && rc == 0; ++compute) {
        int64_t bad = -1;
        rc |= check(ctx, nbx_spots(ctx, &d, compute, NBX_OUT_F32, img, 0, &bad), bad, "nbx_spots");
        if (rc) break;
        /* the same image through a resident plan */
        void* plan = nbx_plan_create(ctx, &d, compute);
        if (!plan) {
            fprintf(stderr, "nbx_plan_create: %s\n", nbx_last_error(ctx));
            rc = 1;
            break;
        }
        rc |= check(ctx, nbx_plan_run(plan, NBX_OUT_F32, again, 0, &bad), bad, "nbx_plan_run");
        nbx_plan_info_t info;
        nbx_plan_info(plan, &info);
        nbx_plan_destroy(plan);
        double total = 0.0;
        int64_t mismatches = 0;
        for (int64_t i = 0; i < n; ++i) {
            total += img[i];
            mismatches += img[i] != again[i];
        }
        char path[4096];
        snprintf(path, sizeof path, "%s.%s.f32", prefix, names[compute]);
        FILE* f = fopen(path, "wb");
        if (!f || fwrite(img, sizeof(float), (size_t)n, f) != (size_t)n) rc = 1;
        if (f) fclose(f);
        printf("%s: %lld pixels, total %.9e photons, kernel variant %d, plan re-run mismatches %lld\n",
               names[compute], (long long)n, total, info.kernel_variant, (long long)mismatches);
        if (mismatches) rc = 1;
    }
    free(img);
    free(again);
    nbx_ctx_destroy(ctx);
    return rc;
}
