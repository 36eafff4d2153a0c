/*
 * nbx.h -- C ABI of the B200-native nanoBragg spot simulator.
 *
 * This is the drop-in boundary for the reference's spot path
 * (xtrace.kernels.nanobragg_spots, /root/reference/pkg/src/xtrace/kernels.py:219-276).
 * The Python host layer (paper_2205_07976_b200/_native.py) binds it with
 * ctypes, which releases the GIL for the duration of every call.
 *
 * Conventions
 *   - Plain C types only: pointers, sizes, doubles.  No torch, no C++ types.
 *   - Every array in a descriptor is caller-owned HOST memory, read (and for
 *     the plan API copied to the device) during the call; nothing is retained.
 *   - Output buffers are caller-owned; `out_on_device` says whether `out` is a
 *     device pointer (on the context's device) or a host pointer.
 *   - Nothing throws across the ABI.  Every entry point returns an NBX_* status;
 *     the message of the last failure is nbx_last_error(ctx).
 *   - One context per GPU; a context (and the plans made from it) must be used
 *     from one host thread at a time.
 *
 * Reference interfaces each entry point replaces are cited per function.
 */
#ifndef NBX_H
#define NBX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NBX_VERSION 10000 /* 1.0.0 */

/* Status codes.  NBX_ERR_ARG mirrors ShapeMismatchError / ValueError
 * (kernels.py:204-208), NBX_ERR_NUMERICAL mirrors NumericalFault wrapped in
 * PatternFault (kernels.py:211-216, execution.py:183-185), NBX_ERR_IO a file that could
 * not be written (CampaignIOError, errors.py:55-61). */
enum {
    NBX_OK = 0,
    NBX_ERR_ARG = 1,
    NBX_ERR_NUMERICAL = 2,
    NBX_ERR_CUDA = 3,
    NBX_ERR_IO = 4
};

/* Arithmetic path of the per-step evaluation. */
enum {
    NBX_COMPUTE_FP64 = 0, /* FP64 everywhere; parity 1e-9 vs the reference's FP64 math */
    NBX_COMPUTE_FP32 = 1  /* FP64 geometry + FP64-exact phase split, FP32 sin/ratio; parity 1e-4 */
};

/* Output modes (what the fused epilogue writes per pixel). */
enum {
    NBX_OUT_F32 = 0,     /* out[p] = f32(scale*acc); the reference store (kernels.py:271-273) */
    NBX_OUT_F64 = 1,     /* out[p] = scale*acc in f64 (extension; the reference rejects f64) */
    NBX_OUT_ADD_F64 = 2, /* out[p] += f64(f32(scale*acc)): spots fused with add_array
                            (kernels.py:315-331, scheduler.py:169-174) */
    NBX_OUT_RAW_F64 = 3, /* out[p] += acc (unscaled FP64 partial, for channel shards) */
    NBX_OUT_IMAGE_F64 = 4, /* out[p] = f64(f32(spots)) + f64(f32(background)): the simulate_image
                              accumulator (scheduler.py:156-183) in one launch; background only when
                              the descriptor carries a profile (bg_points > 0) */
    NBX_OUT_IMAGE_F32 = 5, /* out[p] = f32(IMAGE_F64 value): the write_image payload (io.py:403-434) */
    NBX_OUT_RAW_STORE_F64 = 6 /* out[p] = acc (unscaled partial, plain store): a channel shard written
                                 straight into the root's slot over peer memory (nbx_ipc_*) */
};

/* Lattice shape transforms.  SINCG is the reference's grating
 * (kernels.py:115-142); the others follow the public nanoBragg definitions. */
enum {
    NBX_SHAPE_SINCG = 0,
    NBX_SHAPE_GAUSS = 1,
    NBX_SHAPE_ROUND = 2,
    NBX_SHAPE_TOPHAT = 3
};

/* One rectangular pixel grid -- xtrace.model.DetectorPanel (model.py:328-371)
 * plus the detector-thickness extension. */
typedef struct nbx_panel {
    int32_t slow_pixels;
    int32_t fast_pixels;
    int32_t thick_steps;         /* >= 1; 1 with thickness == 0 reproduces the reference */
    int32_t reserved0;
    double pixel_size;           /* m */
    double distance;             /* m, sample to panel along the beam */
    double beam_center[2];       /* (slow, fast) pixel coordinate of the direct beam */
    double fast_axis[3];         /* unit */
    double slow_axis[3];         /* unit, orthogonal to fast_axis */
    double thickness;            /* m; 0 = infinitely thin sensor (reference semantics) */
    double attenuation_length;   /* m; sensor absorption length (used when thickness > 0) */
} nbx_panel;

/* Everything one spot image needs -- the flattened SpotsContext
 * (kernels.py:100-112) with CrystalModel (model.py:301-325),
 * BeamSpectrum (model.py:374-406) and the panels. */
typedef struct nbx_spots_desc {
    /* detector */
    int32_t n_panels;
    int32_t oversample;          /* sub-pixel grid edge, >= 1 (kernels.py:169) */
    const nbx_panel* panels;     /* n_panels; output is the panels' pixels concatenated */
    /* beam */
    double beam_direction[3];    /* unit */
    int32_t polarization_on;
    int32_t n_sources;
    const double* wavelengths;   /* n_sources, Angstrom, > 0 */
    const double* weights;       /* n_sources, >= 0 */
    double fluence;              /* photons / m^2 */
    double r_e_sqr;              /* m^2, the spot stage; the background stage always uses the
                                    reference module constant R_E_SQR (kernels.py:44,299) */
    /* crystal */
    int32_t n_domains;           /* mosaic domains x phi steps */
    int32_t shape;               /* NBX_SHAPE_* */
    const double* bases;         /* n_domains x 3 x 3, rows a,b,c (Angstrom), already
                                    rotated: CrystalModel.rotated_real_bases (model.py:317-325) */
    int32_t n_cells[3];          /* Na, Nb, Nc >= 1 */
    int32_t n_entries;
    const int32_t* hkl;          /* n_entries x 3 Miller triples */
    const double* amplitudes;    /* n_entries, finite, >= 0 */
    double default_f;            /* amplitude of absent triples (model.py:264-279) */
    /* normalisation: <= 0 means sum(weights) * n_domains * oversample^2
     * (kernels.py:243-245); shards pass the GLOBAL value. */
    double norm;
    /* channel shard: evaluate sources [src_begin, src_end); src_end <= 0 -> all */
    int32_t src_begin;
    int32_t src_end;
    /* diffuse background (add_background, kernels.py:279-312): BackgroundProfile points
     * (stol strictly increasing, 1/Angstrom; amplitudes), used by nbx_background and by
     * NBX_OUT_IMAGE_F64.  bg_points = 0: no background. */
    int32_t bg_points;
    int32_t reserved1;
    const double* bg_stol;
    const double* bg_f;
    double bg_thickness_factor;
} nbx_spots_desc;

/* Filled by nbx_plan_info. */
typedef struct nbx_plan_info_t {
    int64_t n_pixels;            /* output elements */
    int64_t steps;               /* pixel x subpixel x thickness x source x domain */
    int64_t table_cells;         /* dense Fhkl grid cells resident in HBM */
    int32_t table_lo[3];         /* grid origin (h, k, l) */
    int32_t table_dim[3];        /* grid extent */
    int32_t compute;             /* NBX_COMPUTE_* */
    int32_t table_kind;          /* 0 dense grid (magic index), 1 dense grid (wide index) */
    double scale;                /* r_e^2 * fluence / norm */
    int32_t channel_runs;        /* FP64 path: uniform 1/lambda runs evaluated by the channel
                                    recurrence (0: direct per-channel evaluation) */
    int32_t kernel_variant;      /* 0 FP64 direct, 6 FP64 segmented recurrence, 4 FP64 bracket
                                    recurrence (NBX_FP64_REC=1), 1 FP32 MUFU numerator,
                                    5 FP32 polynomial numerator, 2 FP32 degree-4 polynomial */
} nbx_plan_info_t;

int nbx_version(void);

/* sizeof the ABI structs as compiled into the library, for bindings to check their
 * mirrors: 0 nbx_panel, 1 nbx_spots_desc, 2 nbx_plan_info_t (0 for anything else). */
int64_t nbx_struct_size(int which);

/* Number of CUDA devices visible to this process (0 without a GPU or driver). */
int nbx_device_count(void);

/* Per-device context: stream, scratch, last error.  NULL on failure (no GPU). */
void* nbx_ctx_create(int device);
void nbx_ctx_destroy(void* ctx);
const char* nbx_last_error(void* ctx);
/* Launch on a caller stream (cudaStream_t as void*); NULL restores the ctx stream. */
int nbx_ctx_set_stream(void* ctx, void* stream);
int nbx_ctx_synchronize(void* ctx);

/* Output elements a descriptor produces (sum of panel pixels); -1 if invalid. */
int64_t nbx_output_pixels(const nbx_spots_desc* d);

/* One-shot spot image: replaces nanobragg_spots(ctx, out) (kernels.py:219-276).
 * first_bad (may be NULL) receives the lowest non-finite pixel or -1; on a
 * fault the status is NBX_ERR_NUMERICAL and the output is unspecified, as in
 * the reference (execution.py:217-224). */
int nbx_spots(void* ctx, const nbx_spots_desc* d, int compute, int out_mode,
              void* out, int out_on_device, int64_t* first_bad);
/* With NBX_OUT_IMAGE_F64 a fault can come from either stage: *first_bad is the
 * spot stage's lowest bad pixel if any, else the background's, and
 * nbx_fault_stage(ctx) says which (0 spots, 1 background, 2 the f32 downcast of
 * NBX_OUT_IMAGE_F32, i.e. write_image's refusal, io.py:409-411). */
int nbx_fault_stage(void* ctx);

/* Batch of independent images (SURVEY §8 E1 image sharding, config C3; the per-rank
 * image loop of run_campaign, scheduler.py:190-247): outs[i] receives image i; images
 * share nothing.  Each image is one nbx_spots call, so a host `out` is downloaded in row
 * bands overlapping that image's own computation. */
int nbx_spots_batch(void* ctx, const nbx_spots_desc* descs, int n_images, int compute,
                    int out_mode, void* const* outs, int out_on_device, int64_t* first_bad);

/* Plan API: upload a descriptor once (tables, bases, channels resident in
 * HBM), then run it any number of times -- the device analogue of the reference's
 * per-panel geometry cache (_panel_geometry's lru_cache, kernels.py:158). */
void* nbx_plan_create(void* ctx, const nbx_spots_desc* d, int compute);
int nbx_plan_run(void* plan, int out_mode, void* out, int out_on_device, int64_t* first_bad);
int nbx_plan_info(void* plan, nbx_plan_info_t* info);
/* Device-time of the last nbx_plan_run spot kernel (ms, CUDA events). */
double nbx_plan_last_kernel_ms(void* plan);
void nbx_plan_destroy(void* plan);

/* Pipelined image campaign (run_campaign/_rank_task, scheduler.py:190-247,
 * write_image io.py:403-434): image i of descs is rendered as NBX_OUT_IMAGE_F32 and its raw
 * little-endian float32 payload written to paths[i]; crcs[i] receives zlib.crc32 of the payload
 * (the caller writes the JSON sidecar).  The kernel of image i+1 runs while image i is copied
 * to the host, checksummed and written.  image_fault[i] (n_images entries) reports each image:
 *   -1                  written (crcs[i] valid);
 *   (0 << 40) | pixel   non-finite spot pixel, (1 << 40) | pixel non-finite background pixel:
 *                       the image is FLAGGED and skipped and the campaign continues (the
 *                       reference's _rank_task catches the fault and flags it, scheduler.py:212);
 *   (2 << 40) | pixel   the f32 payload is non-finite (write_image refuses it, io.py:409-411; in
 *                       the reference this aborts the rank): the campaign stops, NBX_ERR_NUMERICAL;
 *   -3                  the file could not be written: the campaign stops, NBX_ERR_IO (the
 *                       reference's CampaignIOError, scheduler.py:219-225);
 *   -2                  not run (after a stop).
 * Returns NBX_OK when every image was either written or flagged. */
int nbx_campaign(void* ctx, const nbx_spots_desc* descs, int n_images, int compute,
                 const char* const* paths, uint32_t* crcs, int64_t* image_fault);

/* Image statistics over n values (dtype 0 f32, 1 f64): out = {min, max, mean, total}
 * (image_stats, kernels.py:346-371), the total bit for bit the reference's: NumPy's
 * pairwise sum inside each 8192-value block, parallel_reduce's power-of-two tree across
 * blocks (execution.py:227-285).  n >= 1. */
int nbx_image_stats(void* ctx, const void* data, int64_t n, int dtype, int on_device, double* out4);

/* Histogram (image_histogram, kernels.py:386-430): counts[n_bins] for [lo, hi] with the top
 * bin closed, plus underflow / overflow.  The cumulative counts are the caller's prefix sum. */
int nbx_image_histogram(void* ctx, const void* data, int64_t n, int dtype, int on_device, int n_bins,
                        double lo, double hi, int64_t* counts, int64_t* underflow, int64_t* overflow);

/* zlib-compatible CRC-32 (crc32(crc, data, n)); crc = 0 to start. */
uint32_t nbx_crc32(uint32_t crc, const void* data, int64_t n);

/* Diffuse background image alone -- add_background(profile, panel, spectrum,
 * thickness_factor, out) (kernels.py:279-312): pixel centres, one interpolated
 * f_bg(sin(theta)/lambda)^2 per source.  out_mode NBX_OUT_F32 (the reference's
 * store) / NBX_OUT_F64 / NBX_OUT_ADD_F64 (+= f64(f32), add_array fused).
 * Only panels, beam, spectrum, fluence and the bg_* fields are read (the scale uses the
 * reference constant R_E_SQR, kernels.py:299, not d->r_e_sqr). */
int nbx_background(void* ctx, const nbx_spots_desc* d, int out_mode, void* out, int out_on_device,
                   int64_t* first_bad);

/* Scale + store a reduced raw FP64 image (root of a channel-sharded image,
 * SURVEY §8 E1): out = mode(scale * raw), mode F32, F64 or ADD_F64.  raw is a device
 * pointer. */
int nbx_finalize(void* ctx, const double* raw, int64_t n, double scale, int out_mode,
                 void* out, int out_on_device, int64_t* first_bad);

/* Fused channel-shard transport over peer memory, the alternative
 * to a separate NCCL reduce: the root allocates one FP64 slot per rank in IPC-shareable
 * memory (nbx_ipc_alloc), every other rank maps it (nbx_ipc_open) and its spot kernel's
 * epilogue stores its partial straight into its slot (NBX_OUT_RAW_STORE_F64) -- the transfer
 * happens pixel by pixel while the image is computed -- and after a barrier the root sums
 * the slots in rank order, scales and stores (nbx_reduce_slots).  handle is 64 bytes. */
int nbx_ipc_alloc(void* ctx, int64_t bytes, void** dev, unsigned char* handle);
int nbx_ipc_free(void* ctx, void* dev);
int nbx_ipc_open(void* ctx, const unsigned char* handle, void** dev);
int nbx_ipc_close(void* ctx, void* dev);
/* out = mode(scale * sum_{r < n_slots} slots[r*n + p]), summed in rank order (deterministic). */
int nbx_reduce_slots(void* ctx, const double* slots, int n_slots, int64_t n, double scale, int out_mode,
                     void* out, int out_on_device, int64_t* first_bad);

/* One image split by energy channel over the ranks of a caller's NCCL communicator (SURVEY §8
 * E1, config C5; the north star's "energy-channel shards summed with an NCCL reduce"): every
 * rank calls it with the SAME descriptor (the whole spectrum); rank r evaluates its contiguous
 * source shard (sizes within one, scheduler.py:138-153 plan_batches) into an unscaled FP64
 * partial with the global normalisation (kernels.py:243-245), the partials are summed in place
 * by ncclReduce(ncclFloat64, ncclSum) to `root` on the context's stream, and the root scales
 * and stores the image (out_mode F32 / F64 / ADD_F64, as nbx_finalize; other ranks may pass
 * out = NULL).  nccl_comm is an ncclComm_t; NCCL is resolved from the library already loaded
 * in the process (the one that created the communicator), libnbx does not link it.  Returns
 * after the reduce completed on this rank's stream. */
int nbx_spots_reduce(void* ctx, const nbx_spots_desc* d, int compute, void* nccl_comm, int root,
                     int out_mode, void* out, int out_on_device, int64_t* first_bad);

/* lhs[j] += (double) rhs[j] -- add_array (kernels.py:315-331). */
int nbx_add_array(void* ctx, double* lhs, const float* rhs, int64_t n, int on_device);

/* Poisson photon noise, bit-exact with the host twin nbx_poisson_host
 * (SURVEY §8 X4): out[p] = Poisson(mean[p]) drawn from Philox4x32-10 keyed by
 * (seed, image), counter = p.  mean/out are f64/f32 per `dtype` (0 f32, 1 f64). */
int nbx_add_noise(void* ctx, const void* mean, void* out, int64_t n, int dtype,
                  uint64_t seed, uint64_t image, int on_device);
/* CPU twin of the same sampler (identical bits). */
int nbx_poisson_host(const void* mean, void* out, int64_t n, int dtype,
                     uint64_t seed, uint64_t image);

/* Measurement utility (roofline denominator; MEASURED_PEAKS.json has no FP32/FP64
 * figure): dense FMA throughput of this GPU in TFLOP/s (FMA = 2 FLOP), fp64 = 0
 * for FP32 FFMA, 1 for FP64 DFMA.  Runs ~50-100 ms of independent FMA chains on
 * every SM. */
int nbx_probe_fma_peak(void* ctx, int fp64, double* tflops);

#ifdef __cplusplus
}
#endif

#endif /* NBX_H */
