// nbx_runtime.cu -- host runtime behind the C ABI in include/nbx.h.
//
// Owns: per-device contexts (streams, events, scratch), plan construction
// (validation with the reference's error contract, the dense Fhkl grid sized
// to the reachable Miller box, FP32 range scaling, channel/domain packing,
// HBM upload) and the launches.  Nothing here throws across the ABI: every
// entry point catches and converts to an NBX_* status + last-error string.
#include <cuda_runtime.h>

#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <mutex>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/nbx.h"
#include "nbx_kernels.cuh"
#include "nbx_poisson.h"

namespace nbx {
cudaError_t launch_spots(const SpotsParams& P, int compute, int shape, int idx, cudaStream_t st);
size_t seg_f64_smem_bytes(int n_src, int n_runs);
cudaError_t launch_reduce_slots(const double* slots, int n_slots, int64_t n, double scale, int mode, void* out,
                                unsigned long long* fault, cudaStream_t st);
cudaError_t launch_finalize(const double* raw, int64_t n, double scale, int mode, void* out,
                            unsigned long long* fault, cudaStream_t st);
cudaError_t launch_add_array(double* lhs, const float* rhs, int64_t n, cudaStream_t st);
cudaError_t launch_noise(const void* mean, void* out, int64_t n, int dtype, uint64_t seed, uint64_t image,
                         cudaStream_t st);
cudaError_t launch_fma_probe(int fp64, void* out, int iters, int blocks, cudaStream_t st);
cudaError_t launch_background(const SpotsParams& P, cudaStream_t st);
cudaError_t launch_stats(const void* data, int64_t n, int dtype, void* parts, double* out, cudaStream_t st);
size_t stats_scratch_bytes(int64_t n);
cudaError_t launch_histogram(const void* data, int64_t n, int dtype, int n_bins, double lo, double hi,
                             unsigned long long* counts, cudaStream_t st);
}  // namespace nbx

namespace {

struct ArgError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define NBX_CUDA(call)                                                                         \
    do {                                                                                       \
        cudaError_t e_ = (call);                                                               \
        if (e_ != cudaSuccess)                                                                 \
            throw CudaError(std::string(#call) + ": " + cudaGetErrorString(e_));               \
    } while (0)

// Pinned host staging buffer (grown, never shrunk) for table uploads.
struct HostBuf {
    void* p = nullptr;
    size_t bytes = 0;
    HostBuf() = default;
    HostBuf(const HostBuf&) = delete;
    HostBuf& operator=(const HostBuf&) = delete;
    ~HostBuf() { release(); }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        bytes = 0;
    }
    template <typename T>
    T* ensure(size_t n) {
        if (n * sizeof(T) > bytes) {
            release();
            NBX_CUDA(cudaHostAlloc(&p, n * sizeof(T), cudaHostAllocDefault));
            bytes = n * sizeof(T);
        }
        return static_cast<T*>(p);
    }
};

// Device buffer that frees itself (grown, never shrunk).
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    void ensure(size_t n) {
        if (n <= bytes) return;
        release();
        NBX_CUDA(cudaMalloc(&p, n));
        bytes = n;
    }
};

struct Plan;

struct Ctx {
    int device = 0;
    int fault_stage = 0;      // stage of the last reported fault: 0 spots, 1 background, 2 downcast
    // campaign pipeline: second stream (device-to-host copies) and double buffers
    cudaStream_t copy_stream = nullptr;
    Plan* camp_plan[2] = {nullptr, nullptr};
    DevBuf camp_out[2], camp_fault[2];
    void* camp_host[2] = {nullptr, nullptr};
    unsigned long long* camp_fault_host = nullptr;  // pinned [2][kFaultSlots]
    size_t camp_host_bytes = 0;
    Plan* oneshot = nullptr;  // device buffers reused by nbx_spots (cudaFree can stall for ~100 ms)
    cudaStream_t own = nullptr;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // pipelined host-output runs: a second compute stream (row bands alternate so
    // one band's tail overlaps the next band's head) and one event per band
    cudaStream_t stream2 = nullptr;
    cudaEvent_t band_ev[16] = {};
    cudaEvent_t join_ev = nullptr;
    DevBuf out_scratch;     // device image when the caller passes host memory
    DevBuf stage_in, stats_parts, stats_res, hist_counts;  // image_stats / image_histogram scratch
    DevBuf raw_scratch;     // FP64 partial of a long spectrum split into channel shards
    DevBuf img_scratch;     // simulate_image accumulator of a long spectrum (device, f64)
    DevBuf fault;           // one u64
    std::string err;
};

// Device copies of the background profile and the {lambda, w} table it needs.
struct BgBufs {
    DevBuf chan, stol, f;
};

struct Plan {
    Ctx* ctx = nullptr;
    int compute = 0;
    int kernel_variant = 0;  // 0 FP64, 1 FP32 (MUFU numerator), 2 FP32 with the degree-4 polynomial
                             // (NBX_FP32_POLY=4), 5 FP32 degree 3 with the polynomial numerator,
                             // 4 FP64 bracket recurrence, 6 FP64 segmented recurrence,
                             // 7 FP32 MUFU numerator with segmented indices (uniform spectra)
    int shape = 0;
    bool wide = false;        // dense grid with integer index (FP32 magic window exceeded)
    bool hash = false;        // sparse Fhkl table (reachable box above kDenseMaxCells)
    cudaTextureObject_t tex = 0;  // texture view of `table` (FP32 power-of-two grid)
    const void* tex_ptr = nullptr;
    size_t tex_bytes = 0;
    void release_tex() {
        if (tex) cudaDestroyTextureObject(tex);
        tex = 0;
        tex_ptr = nullptr;
        tex_bytes = 0;
    }
    ~Plan() { release_tex(); }
    DevBuf hkeys, hvals;
    nbx::SpotsParams P{};
    DevBuf panels, bases, chan, chunks, table, runs, chunk_step;
    HostBuf host_table;       // pinned staging of the F^2 grid
    // The device F^2 grid is rebuilt only when its inputs change: consecutive images of one
    // crystal (new orientation / mosaic / spectrum jitter) share the table, so a re-used plan
    // (nbx_spots' one-shot plan, the campaign's two) skips the fill, validation and upload.
    struct TableKey {
        bool valid = false;
        int compute = -1;
        int hmax[3] = {0, 0, 0};
        int32_t sH = 0, sK = 0;
        double default_f = 0.0, sigma = 0.0, maxf2 = 0.0;
        const void* dev = nullptr;
        std::vector<int32_t> hkl;
        std::vector<double> amp;
    } tkey;
    BgBufs bg;
    bool uniform_panels = true;  // every panel has the same (slow, fast): row bands are 2-D copies
    int64_t n_pixels = 0;
    int64_t steps = 0;
    nbx_plan_info_t info{};
    double scale = 0.0;      // r_e^2 fluence / norm
    double out_scale = 0.0;  // scale / sigma
    float last_ms = -1.f;
    bool timed = false;
};

// --------------------------------------------------------------------------
// Validation: mirrors the reference's constructors and kernel checks
// (model.py:328-406, kernels.py:204-208) so the same bad inputs fail.
// --------------------------------------------------------------------------
bool finite(double x) { return std::isfinite(x); }

bool trace_enabled() {
    static const bool on = [] {
        const char* v = std::getenv("NBX_TRACE");
        return v != nullptr && *v != '\0' && std::strcmp(v, "0") != 0;
    }();
    return on;
}

// NVTX ranges (the reference's kernel_timer labels, execution.py:350-356, as
// profiler ranges): plan build, launch, download, campaign write-out.  Header-only NVTX v3:
// no cost unless a profiler (nsys / ncu --nvtx) is attached.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

constexpr double kReSqr = 7.94079248e-30;  // classical electron radius squared, m^2 (kernels.py:44)

double norm3(const double* v) { return std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]); }

void check_unit(const double* v, const char* what) {
    for (int i = 0; i < 3; ++i)
        if (!finite(v[i])) throw ArgError(std::string(what) + " must be finite");
    if (std::fabs(norm3(v) - 1.0) > 1e-12) throw ArgError(std::string(what) + " must be a unit vector");
}

int64_t count_pixels(const nbx_spots_desc* d) {
    if (!d || d->n_panels < 1 || !d->panels) throw ArgError("descriptor needs at least one panel");
    int64_t n = 0;
    for (int i = 0; i < d->n_panels; ++i) {
        const nbx_panel& p = d->panels[i];
        if (p.slow_pixels < 1 || p.fast_pixels < 1) throw ArgError("panel must have at least one pixel per axis");
        n += (int64_t)p.slow_pixels * p.fast_pixels;
    }
    return n;
}

void validate(const nbx_spots_desc* d) {
    count_pixels(d);
    if (d->oversample < 1) throw ArgError("oversample must be >= 1");
    for (int i = 0; i < d->n_panels; ++i) {
        const nbx_panel& p = d->panels[i];
        if (!(p.pixel_size > 0) || !finite(p.pixel_size)) throw ArgError("pixel_size must be > 0");
        if (!(p.distance > 0) || !finite(p.distance)) throw ArgError("distance must be > 0");
        if (!finite(p.beam_center[0]) || !finite(p.beam_center[1])) throw ArgError("beam_center must be finite");
        check_unit(p.fast_axis, "fast_axis");
        check_unit(p.slow_axis, "slow_axis");
        const double dot = p.fast_axis[0] * p.slow_axis[0] + p.fast_axis[1] * p.slow_axis[1] +
                           p.fast_axis[2] * p.slow_axis[2];
        if (std::fabs(dot) > 1e-12) throw ArgError("fast_axis and slow_axis must be orthogonal");
        if (p.thick_steps < 1) throw ArgError("thick_steps must be >= 1");
        if (!(p.thickness >= 0) || !finite(p.thickness)) throw ArgError("thickness must be finite and >= 0");
        if (p.thickness > 0 && !(p.attenuation_length > 0 && finite(p.attenuation_length)))
            throw ArgError("attenuation_length must be > 0 when thickness > 0");
    }
    check_unit(d->beam_direction, "beam_direction");
    if (d->n_sources < 1 || !d->wavelengths || !d->weights)
        throw ArgError("spectrum needs at least one wavelength sample");
    bool any_pos = false;
    for (int i = 0; i < d->n_sources; ++i) {
        if (!(d->wavelengths[i] > 0) || !finite(d->wavelengths[i])) throw ArgError("wavelengths must be > 0");
        if (!finite(d->weights[i]) || d->weights[i] < 0) throw ArgError("weights must be finite and >= 0");
        any_pos |= d->weights[i] > 0;
    }
    if (!any_pos && !(d->norm > 0)) throw ArgError("at least one sample must have weight > 0");
    if (!finite(d->fluence) || d->fluence < 0) throw ArgError("fluence must be finite and >= 0");
    if (!finite(d->r_e_sqr)) throw ArgError("r_e_sqr must be finite");
    if (d->n_domains < 1 || !d->bases) throw ArgError("mosaic rotations must be a non-empty (n, 3, 3) array");
    for (int i = 0; i < 9 * d->n_domains; ++i)
        if (!finite(d->bases[i])) throw ArgError("rotated bases must be finite");
    for (int a = 0; a < 3; ++a)
        if (d->n_cells[a] < 1) throw ArgError("n_cells must all be >= 1");
    if (d->shape < 0 || d->shape > 3) throw ArgError("unknown shape transform");
    if (d->n_entries < 0 || (d->n_entries > 0 && (!d->hkl || !d->amplitudes)))
        throw ArgError("structure-factor table arrays missing");
    if (!finite(d->default_f) || d->default_f < 0) throw ArgError("default_f must be finite and non-negative");
    const int sb = d->src_begin, se = d->src_end <= 0 ? d->n_sources : d->src_end;
    if (sb < 0 || se > d->n_sources || sb >= se) throw ArgError("invalid source shard range");
}

void validate_entries(const nbx_spots_desc* d) {
    for (int i = 0; i < d->n_entries; ++i) {
        const double f = d->amplitudes[i];
        if (!finite(f) || f < 0) throw ArgError("amplitudes must be finite and >= 0");
        for (int a = 0; a < 3; ++a)
            if (std::abs((int64_t)d->hkl[3 * i + a]) >= (1 << 20)) throw ArgError("Miller index out of supported range");
    }
}

// Largest |s_out - beam| over every sub-pixel / layer position of every panel.
// The set {x : angle(x, beam) <= alpha} is a convex cone for alpha < 90 deg, so
// the maximum over a (slab of a) rectangle is attained at one of its corners.
double max_rel(const nbx_spots_desc* d) {
    const double* b = d->beam_direction;
    double min_cos = 1.0;
    for (int i = 0; i < d->n_panels; ++i) {
        const nbx_panel& p = d->panels[i];
        double nrm[3] = {p.fast_axis[1] * p.slow_axis[2] - p.fast_axis[2] * p.slow_axis[1],
                         p.fast_axis[2] * p.slow_axis[0] - p.fast_axis[0] * p.slow_axis[2],
                         p.fast_axis[0] * p.slow_axis[1] - p.fast_axis[1] * p.slow_axis[0]};
        const double sgn = (nrm[0] * b[0] + nrm[1] * b[1] + nrm[2] * b[2]) < 0 ? -1.0 : 1.0;
        const double depth_max = p.thickness > 0 ? p.thickness : 0.0;
        for (int c = 0; c < 8; ++c) {
            const double s = ((c & 1) ? (double)p.slow_pixels : 0.0) - p.beam_center[0];
            const double f = ((c & 2) ? (double)p.fast_pixels : 0.0) - p.beam_center[1];
            const double dep = (c & 4) ? depth_max : 0.0;
            double q[3];
            for (int a = 0; a < 3; ++a)
                q[a] = p.distance * b[a] + s * p.pixel_size * p.slow_axis[a] + f * p.pixel_size * p.fast_axis[a] +
                       dep * sgn * nrm[a];
            const double cs = (q[0] * b[0] + q[1] * b[1] + q[2] * b[2]) / norm3(q);
            min_cos = std::min(min_cos, cs);
        }
    }
    if (min_cos <= 0.02) return 2.0;
    return std::sqrt(std::max(0.0, 2.0 - 2.0 * min_cos)) * (1.0 + 1e-9) + 1e-12;
}

// Per-panel kernel constants (DetectorPanel, model.py:328-371, + the X1 layers).
std::vector<nbx::DevPanel> make_panels(const nbx_spots_desc* d, int* max_slow, int* max_fast, int64_t* n_pix,
                                       int64_t* sub_steps) {
    std::vector<nbx::DevPanel> hp(d->n_panels);
    int64_t off = 0, subs = 0;
    const int os = d->oversample < 1 ? 1 : d->oversample;
    for (int i = 0; i < d->n_panels; ++i) {
        const nbx_panel& s = d->panels[i];
        nbx::DevPanel& t = hp[i];
        std::memset(&t, 0, sizeof(t));
        t.slow = s.slow_pixels;
        t.fast = s.fast_pixels;
        t.out_offset = off;
        t.pixel_size = s.pixel_size;
        t.distance = s.distance;
        t.bc_slow = s.beam_center[0];
        t.bc_fast = s.beam_center[1];
        for (int a = 0; a < 3; ++a) {
            t.fast_axis[a] = s.fast_axis[a];
            t.slow_axis[a] = s.slow_axis[a];
        }
        t.normal[0] = s.fast_axis[1] * s.slow_axis[2] - s.fast_axis[2] * s.slow_axis[1];
        t.normal[1] = s.fast_axis[2] * s.slow_axis[0] - s.fast_axis[0] * s.slow_axis[2];
        t.normal[2] = s.fast_axis[0] * s.slow_axis[1] - s.fast_axis[1] * s.slow_axis[0];
        const double* b = d->beam_direction;
        const double sgn = (t.normal[0] * b[0] + t.normal[1] * b[1] + t.normal[2] * b[2]) < 0 ? -1.0 : 1.0;
        for (int a = 0; a < 3; ++a) t.odet[a] = sgn * t.normal[a];
        if (s.thickness > 0) {
            t.thick_steps = s.thick_steps;
            t.thick_step = s.thickness / (double)s.thick_steps;
            t.inv_atten = 1.0 / s.attenuation_length;
        } else {
            t.thick_steps = 1;  // a thin sensor has exactly one layer (reference)
            t.thick_step = 0.0;
            t.inv_atten = 0.0;
        }
        const int64_t npx = (int64_t)s.slow_pixels * s.fast_pixels;
        off += npx;
        subs += npx * (int64_t)(os * os) * t.thick_steps;
        *max_slow = std::max(*max_slow, s.slow_pixels);
        *max_fast = std::max(*max_fast, s.fast_pixels);
    }
    *n_pix = off;
    *sub_steps = subs;
    return hp;
}

// Background profile checks (BackgroundProfile, model.py:409-435) + device upload.
void setup_background(const nbx_spots_desc* d, nbx::SpotsParams& P, BgBufs& B) {
    P.bg_points = 0;
    if (d->bg_points <= 0) return;
    if (d->bg_points < 2 || !d->bg_stol || !d->bg_f) throw ArgError("background profile needs at least 2 points");
    for (int i = 0; i < d->bg_points; ++i) {
        if (!finite(d->bg_stol[i]) || d->bg_stol[i] < 0) throw ArgError("stol values must be >= 0");
        if (i > 0 && !(d->bg_stol[i] > d->bg_stol[i - 1])) throw ArgError("stol values must be strictly increasing");
        if (!finite(d->bg_f[i]) || d->bg_f[i] < 0) throw ArgError("background amplitudes must be finite and >= 0");
    }
    if (!finite(d->bg_thickness_factor)) throw ArgError("thickness_factor must be finite");
    double wsum = 0.0;
    std::vector<nbx::BgChan> lw(d->n_sources);
    for (int i = 0; i < d->n_sources; ++i) {
        lw[i] = nbx::BgChan{d->wavelengths[i], 1.0 / d->wavelengths[i], d->weights[i], 0.0};
        wsum += d->weights[i];
    }
    B.chan.ensure(lw.size() * sizeof(nbx::BgChan));
    NBX_CUDA(cudaMemcpy(B.chan.p, lw.data(), lw.size() * sizeof(nbx::BgChan), cudaMemcpyHostToDevice));
    // {f_j, slope_j}: np.interp's own precomputed slopes (same IEEE expression)
    std::vector<double> fs(2 * (size_t)d->bg_points, 0.0);
    for (int i = 0; i < d->bg_points; ++i) {
        fs[2 * i] = d->bg_f[i];
        if (i + 1 < d->bg_points)
            fs[2 * i + 1] = (d->bg_f[i + 1] - d->bg_f[i]) / (d->bg_stol[i + 1] - d->bg_stol[i]);
    }
    B.stol.ensure(sizeof(double) * d->bg_points);
    B.f.ensure(sizeof(double) * fs.size());
    NBX_CUDA(cudaMemcpy(B.stol.p, d->bg_stol, sizeof(double) * d->bg_points, cudaMemcpyHostToDevice));
    NBX_CUDA(cudaMemcpy(B.f.p, fs.data(), sizeof(double) * fs.size(), cudaMemcpyHostToDevice));
    P.bg_chan = static_cast<const nbx::BgChan*>(B.chan.p);
    P.bg_stol = static_cast<const double*>(B.stol.p);
    P.bg_fs = static_cast<const double2*>(B.f.p);
    P.n_bg_chan = d->n_sources;
    P.bg_points = d->bg_points;
    // kernels.py:299 uses the module constant R_E_SQR (kernels.py:44), never a context's r_e_sqr:
    // a fused spots + background image keeps the reference's composition even when the spot
    // context carries a non-default r_e_sqr
    P.bg_scale = kReSqr * d->fluence * d->bg_thickness_factor / wsum;
}

// Build (or, with `reuse`, rebuild in place -- its device buffers only grow) a plan.
constexpr int64_t kDenseMaxCells = int64_t(1) << 26;
// Sources per launch (one plan): the channel table, runs and per-thread state of every kernel
// variant fit the shared memory of a block at this size; longer spectra are split into
// channel shards by nbx_spots / nbx_spots_reduce.
constexpr int kMaxShardSources = 8192;

// Sparse Fhkl table (index kind 2): open addressing, linear probing, at most half full;
// the key packing and hash are the kernel's (nbx_kernels.cu:pack_hkl / hash_slot).  A
// repeated (h, k, l) keeps its last amplitude.  Values are F^2 (x sigma on FP32).
uint64_t pack_hkl_host(int h, int k, int l) {
    return ((uint64_t)(uint32_t)(h + (1 << 20)) << 42) | ((uint64_t)(uint32_t)(k + (1 << 20)) << 21) |
           (uint64_t)(uint32_t)(l + (1 << 20));
}

void build_hash(Plan* plan, const nbx_spots_desc* d, int compute, double def2, double sigma) {
    uint64_t size = 1024;
    while (size < 2 * (uint64_t)std::max(d->n_entries, 1)) size <<= 1;
    if (size > (uint64_t(1) << 31)) throw ArgError("structure-factor table too large");
    const uint32_t mask = (uint32_t)(size - 1);
    std::vector<unsigned long long> keys(size, ~0ull);
    std::vector<double> v64(size, 0.0);
    for (int i = 0; i < d->n_entries; ++i) {
        const uint64_t key = pack_hkl_host(d->hkl[3 * i], d->hkl[3 * i + 1], d->hkl[3 * i + 2]);
        uint32_t s = (uint32_t)((key * 0x9E3779B97F4A7C15ull) >> 32) & mask;
        while (keys[s] != ~0ull && keys[s] != key) s = (s + 1) & mask;
        keys[s] = key;
        v64[s] = d->amplitudes[i] * d->amplitudes[i];
    }
    plan->hkeys.ensure(size * sizeof(unsigned long long));
    NBX_CUDA(cudaMemcpy(plan->hkeys.p, keys.data(), size * sizeof(unsigned long long), cudaMemcpyHostToDevice));
    nbx::SpotsParams& P = plan->P;
    if (compute == NBX_COMPUTE_FP32) {
        std::vector<float> v32(size);
        for (uint64_t i = 0; i < size; ++i) v32[i] = (float)(v64[i] * sigma);
        plan->hvals.ensure(size * sizeof(float));
        NBX_CUDA(cudaMemcpy(plan->hvals.p, v32.data(), size * sizeof(float), cudaMemcpyHostToDevice));
    } else {
        plan->hvals.ensure(size * sizeof(double));
        NBX_CUDA(cudaMemcpy(plan->hvals.p, v64.data(), size * sizeof(double), cudaMemcpyHostToDevice));
    }
    P.hash_keys = static_cast<const unsigned long long*>(plan->hkeys.p);
    P.hash_vals = plan->hvals.p;
    P.hash_mask = mask;
    P.hash_def_d = def2;
    P.hash_def_f = (float)(def2 * sigma);
    plan->info.table_cells = (int64_t)size;
}

// NBX_TRACE: wall time of the phases of a plan build, printed to stderr.
struct PhaseTimer {
    bool on = trace_enabled();
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    std::string log;
    void mark(const char* what) {
        if (!on) return;
        const auto n = std::chrono::steady_clock::now();
        char buf[64];
        std::snprintf(buf, sizeof(buf), " %s %.3f", what, std::chrono::duration<double, std::milli>(n - t).count());
        log += buf;
        t = n;
    }
    ~PhaseTimer() {
        if (on && !log.empty()) std::fprintf(stderr, "[nbx] plan ms:%s\n", log.c_str());
    }
};

Plan* build_plan(Ctx* ctx, const nbx_spots_desc* d, int compute, Plan* reuse = nullptr) {
    NvtxRange nvtx("nbx plan build");
    PhaseTimer pt;
    validate(d);
    pt.mark("validate");
    if (compute != NBX_COMPUTE_FP64 && compute != NBX_COMPUTE_FP32) throw ArgError("unknown compute path");
    auto plan = reuse ? reuse : new Plan();
    if (reuse) {
        plan->P = nbx::SpotsParams{};
        plan->info = nbx_plan_info_t{};
        plan->wide = false;
        plan->hash = false;
        plan->last_ms = -1.f;
    }
    try {
        plan->ctx = ctx;
        plan->compute = compute;
        plan->kernel_variant = compute == NBX_COMPUTE_FP32 ? 1 : 0;
        if (compute == NBX_COMPUTE_FP32) {
            const char* ev = std::getenv("NBX_FP32_POLY");
            if (ev && std::atoi(ev) == 4) plan->kernel_variant = 2;
        }
        plan->shape = d->shape;
        nbx::SpotsParams& P = plan->P;
        const int sb = d->src_begin, se = d->src_end <= 0 ? d->n_sources : d->src_end;
        const int n_src = se - sb;
        const int os = d->oversample;

        // normalisation and scale (kernels.py:242-245)
        double norm = d->norm;
        if (!(norm > 0)) {
            double wsum = 0.0;
            for (int i = 0; i < d->n_sources; ++i) wsum += d->weights[i];
            norm = wsum * (double)d->n_domains * (double)(os * os);
        }
        plan->scale = d->r_e_sqr * d->fluence / norm;

        // panels
        int max_slow = 0, max_fast = 0;
        int64_t off = 0, sub_steps = 0;
        const std::vector<nbx::DevPanel> hp = make_panels(d, &max_slow, &max_fast, &off, &sub_steps);
        plan->n_pixels = off;
        plan->steps = sub_steps * (int64_t)n_src * d->n_domains;
        if (plan->kernel_variant == 1 && d->shape == NBX_SHAPE_SINCG) {
            // MUFU.SIN's ~1e-6 absolute error averages out over the many (channel, domain,
            // sub-pixel) samples of a pixel; with few samples per pixel (the C1 toy: one
            // channel x one domain, side lobes sampled one point per pixel) nothing averages,
            // and such images are small: take the degree-4 polynomial loop (variant 2, worst
            // golden margin 83x instead of 9.8x for degree 3).  NBX_FP32_NUM=mufu|poly forces
            // the MUFU loop or the degree-3 polynomial loop (variant 5).
            const char* nev = std::getenv("NBX_FP32_NUM");
            const double per_pixel = off > 0 ? (double)plan->steps / (double)off : 0.0;
            if (per_pixel < 256.0) plan->kernel_variant = 2;
            if (nev && std::strcmp(nev, "mufu") == 0) plan->kernel_variant = 1;
            if (nev && std::strcmp(nev, "poly") == 0) plan->kernel_variant = 5;
        }
        plan->uniform_panels = true;
        for (const auto& q : hp) plan->uniform_panels &= (q.slow == max_slow && q.fast == max_fast);

        // reachable Miller box (+1 margin for rounding) -> dense grid
        const double relmax = max_rel(d);
        double ivmax = 0.0;
        for (int i = sb; i < se; ++i) ivmax = std::max(ivmax, 1.0 / d->wavelengths[i]);
        int hmax[3];
        bool huge = false;
        for (int a = 0; a < 3; ++a) {
            double m = 0.0;
            for (int dd = 0; dd < d->n_domains; ++dd) m = std::max(m, norm3(d->bases + 9 * dd + 3 * a));
            const double hb = std::ceil(m * relmax * ivmax) + 1.0;
            huge |= hb > (double)(1 << 20);
            hmax[a] = (int)std::min(hb, (double)(1 << 20));
        }
        const int64_t dims[3] = {2 * (int64_t)hmax[0] + 1, 2 * (int64_t)hmax[1] + 1, 2 * (int64_t)hmax[2] + 1};
        const int64_t cells = dims[0] * dims[1] * dims[2];
        // Dense grid up to kDenseMaxCells (64M cells: every protein-sized cell at any
        // resolution the detector reaches); beyond it (virus-sized cells) a sparse table.
        const char* hev = std::getenv("NBX_FHKL_HASH");
        plan->hash = huge || cells > kDenseMaxCells || (hev && std::atoi(hev) == 1);
        if (plan->hash && compute == NBX_COMPUTE_FP32) plan->kernel_variant = 5;  // scalar polynomial loop
        for (int a = 0; a < 3; ++a) P.lo[a] = -hmax[a];
        P.sK = (int32_t)dims[2];
        P.sH = (int32_t)(dims[1] * dims[2]);
        int64_t cells_alloc = plan->hash ? 0 : cells;
        plan->wide = false;
        if (compute == NBX_COMPUTE_FP32 && !plan->hash) {
            // FP32 index: power-of-two strides so that the cell number is two shift-adds
            // of the magic-rounded floats' bit patterns (ALU pipe, no FMA-pipe work):
            //   bits(mA) << lg(sH) + bits(mB) << lg(sK) + bits(mC) = cell + c (mod 2^32),
            // c = 0x4B400000 (sH + sK + 1) mod 2^32 absorbed by the base pointer.
            // Needs every cell + offset (|j| <= 2) inside the 2^22 magic window and no
            // 2^32 wrap; otherwise the WIDE (integer-conversion) index is used.
            int lk = 0, lh = 0;
            while ((int64_t(1) << lk) < dims[2]) ++lk;
            while ((int64_t(1) << lh) < dims[1]) ++lh;
            const int64_t sK2 = int64_t(1) << lk, sH2 = int64_t(1) << (lk + lh);
            const int64_t alloc2 = dims[0] * sH2;
            const uint64_t c = (uint64_t(0x4B400000u) * (uint64_t)(sH2 + sK2 + 1)) & 0xFFFFFFFFull;
            if (alloc2 + 2 * (sH2 + sK2 + 1) < (int64_t(1) << 22) && c + (uint64_t)alloc2 < (uint64_t(1) << 32)) {
                P.sK = (int32_t)sK2;
                P.sH = (int32_t)sH2;
                P.sh_k = lk;
                P.sh_h = lk + lh;
                P.lea_bias = (uint32_t)c;
                cells_alloc = alloc2;
            } else {
                plan->wide = true;
            }
        }
        double smax = 0.0;  // largest |rel . a| over domains and axes (Angstrom)
        for (int dd = 0; dd < d->n_domains; ++dd)
            for (int a = 0; a < 3; ++a) smax = std::max(smax, norm3(d->bases + 9 * dd + 3 * a) * relmax);

        pt.mark("geometry");
        // F^2 grid (FP64 exact; FP32 scaled by a power of two sigma), built straight
        // into pinned staging memory: first the largest reachable F^2, then the fill
        const double def2 = d->default_f * d->default_f;
        auto reachable = [&](int i) {
            return plan->hash || (std::abs(d->hkl[3 * i]) <= hmax[0] && std::abs(d->hkl[3 * i + 1]) <= hmax[1] &&
                                  std::abs(d->hkl[3 * i + 2]) <= hmax[2]);
        };
        auto cell_of = [&](int i) {
            return (int64_t)(d->hkl[3 * i] + hmax[0]) * P.sH + (int64_t)(d->hkl[3 * i + 1] + hmax[1]) * P.sK +
                   (d->hkl[3 * i + 2] + hmax[2]);
        };
        Plan::TableKey& tk = plan->tkey;
        const bool same_entries =
            tk.valid && tk.compute == compute && tk.default_f == d->default_f && tk.sH == P.sH && tk.sK == P.sK &&
            tk.hmax[0] == hmax[0] && tk.hmax[1] == hmax[1] && tk.hmax[2] == hmax[2] &&
            tk.hkl.size() == 3 * (size_t)d->n_entries && tk.amp.size() == (size_t)d->n_entries &&
            (d->n_entries == 0 ||
             (std::memcmp(tk.hkl.data(), d->hkl, tk.hkl.size() * sizeof(int32_t)) == 0 &&
              std::memcmp(tk.amp.data(), d->amplitudes, tk.amp.size() * sizeof(double)) == 0));
        double maxf2 = def2;
        if (same_entries) {
            maxf2 = tk.maxf2;
        } else {
            validate_entries(d);
            for (int i = 0; i < d->n_entries; ++i)
                if (reachable(i)) maxf2 = std::max(maxf2, d->amplitudes[i] * d->amplitudes[i]);
        }
        double sigma = 1.0;
        if (compute == NBX_COMPUTE_FP32) {
            double maxw = 0.0;
            for (int i = sb; i < se; ++i) maxw = std::max(maxw, d->weights[i]);
            const double nnn = (double)d->n_cells[0] * d->n_cells[1] * d->n_cells[2];
            const double peak = maxf2 * maxw * nnn * nnn;
            if (peak > 0 && finite(peak)) {
                int e = (int)std::floor(100.0 - std::log2(peak));
                e = std::max(-1000, std::min(e, 100));
                sigma = std::ldexp(1.0, e);
            }
        }
        // device table still current: same entries, grid and scale, buffer not reallocated
        const size_t tbytes = (size_t)cells_alloc * (compute == NBX_COMPUTE_FP32 ? sizeof(float) : sizeof(double));
        const bool table_current = !plan->hash && same_entries && tk.sigma == sigma && tk.dev == plan->table.p &&
                                   plan->table.bytes >= tbytes;
        if (!table_current) tk.valid = false;  // re-armed after the upload below
        if (plan->hash) {
            build_hash(plan, d, compute, def2, sigma);
        } else if (table_current) {
            // nothing to fill or upload
        } else if (compute == NBX_COMPUTE_FP32) {
            float* tf = plan->host_table.ensure<float>(cells_alloc);
            std::fill(tf, tf + cells_alloc, (float)(def2 * sigma));
            for (int i = 0; i < d->n_entries; ++i)
                if (reachable(i)) tf[cell_of(i)] = (float)(d->amplitudes[i] * d->amplitudes[i] * sigma);
        } else {
            double* t64 = plan->host_table.ensure<double>(cells_alloc);
            std::fill(t64, t64 + cells_alloc, def2);
            for (int i = 0; i < d->n_entries; ++i)
                if (reachable(i)) t64[cell_of(i)] = d->amplitudes[i] * d->amplitudes[i];
        }
        plan->out_scale = plan->scale / sigma;
        pt.mark("grid");

        // channels
        int n_chan_entries = n_src;  // FP64: channels; FP32: channel pairs
        if (compute == NBX_COMPUTE_FP32) {
            // sort by 1/lambda and cut chunks whose phase offsets stay small:
            // |S (iv - iv0)| <= smax (max - min) / 2 <= 1 -> |x| <= 1.5 in the kernel
            std::vector<int> order(n_src);
            std::vector<double> iv(n_src);
            for (int i = 0; i < n_src; ++i) {
                order[i] = i;
                iv[i] = 1.0 / d->wavelengths[sb + i];  // kernels.py:257
            }
            std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return iv[x] < iv[y]; });
            // pairs {D_w, D_w+1, wt_w, wt_w+1} for the packed (f32x2) loop; an odd
            // chunk is padded with a zero-weight copy of its last channel
            std::vector<nbx::ChunkF32> chunks;
            std::vector<float> ch;
            // Segmented FP32 MUFU loop (variant 7): chunks of a uniform spectrum cut so that every
            // reachable phase spans <= 0.9 over a chunk (at most one index change per axis), the
            // chunk's 1/lambda step handed to the kernel for the crossing prediction.
            // Opt-in (NBX_FP32_SEG=1): on C2 it is 116 ms against the per-channel loop's 110 ms --
            // ~8 warp stops per 50-pair chunk cost what the 17 saved instructions per pair gain,
            // and with 34 FMA lane-ops per channel the four MUFUs per channel co-limit.
            const char* sev = std::getenv("NBX_FP32_SEG");
            bool seg32 = plan->kernel_variant == 1 && d->shape == NBX_SHAPE_SINCG && !plan->hash && sev &&
                         std::atoi(sev) == 1;
            std::vector<float> chunk_step;
            const double half_lim = seg32 ? 0.45 : 1.0;
            // Chunks hold <= kChunkMax channels (the FP32 partial of each packed half sums
            // <= 64 terms) and a phase-feasible run of L channels is cut into ceil(L / max)
            // chunks of equal size (C2's 100 channels: one chunk; 130: 66 + 64, not 128 + 2).
            int i0 = 0, npairs = 0;
            const char* cev = std::getenv("NBX_CHUNK_MAX");
            const int chunk_max = cev ? std::max(2, std::atoi(cev)) : 128;
            int run_end = 0, run_chunk = chunk_max;
            while (i0 < n_src) {
                if (i0 >= run_end) {  // next phase-feasible run and its balanced chunk size
                    run_end = i0 + 1;
                    while (run_end < n_src && (iv[order[run_end]] - iv[order[i0]]) * 0.5 * smax <= half_lim) ++run_end;
                    const int len = run_end - i0, k = (len + chunk_max - 1) / chunk_max;
                    run_chunk = std::min(chunk_max, ((len + k - 1) / k + 1) / 2 * 2);  // even: whole pairs
                }
                const int i1 = std::min(run_end, i0 + run_chunk);
                const double iv0 = 0.5 * (iv[order[i0]] + iv[order[i1 - 1]]);
                const int p0 = npairs;
                for (int q = i0; q < i1; q += 2) {
                    const int q1 = q + 1 < i1 ? q + 1 : q;
                    ch.push_back((float)(iv[order[q]] - iv0));
                    ch.push_back((float)(iv[order[q1]] - iv0));
                    ch.push_back((float)d->weights[sb + order[q]]);
                    ch.push_back(q + 1 < i1 ? (float)d->weights[sb + order[q1]] : 0.0f);
                    ++npairs;
                }
                chunks.push_back(nbx::ChunkF32{iv0, p0, npairs});
                if (seg32) {  // uniform to 1e-7 of phase for every reachable S (the prediction's budget)
                    const int len = i1 - i0;
                    const double delta = len > 1 ? (iv[order[i1 - 1]] - iv[order[i0]]) / (double)(len - 1) : 0.0;
                    double dev = 0.0;
                    for (int k = 0; k < len; ++k)
                        dev = std::max(dev, std::fabs(iv[order[i0 + k]] - iv[order[i0]] - (double)k * delta));
                    if (dev * smax > 1e-7) seg32 = false;
                    chunk_step.push_back((float)delta);
                }
                i0 = i1;
            }
            if (seg32 && (int64_t)chunks.size() * 8 > n_src) seg32 = false;  // chunks too short to pay off
            if (seg32) {
                plan->kernel_variant = 7;
                plan->chunk_step.ensure(chunk_step.size() * sizeof(float));
                NBX_CUDA(cudaMemcpy(plan->chunk_step.p, chunk_step.data(), chunk_step.size() * sizeof(float),
                                    cudaMemcpyHostToDevice));
                P.chunk_step = static_cast<const float*>(plan->chunk_step.p);
            }
            n_chan_entries = npairs;
            plan->chan.ensure(ch.size() * sizeof(float));
            NBX_CUDA(cudaMemcpy(plan->chan.p, ch.data(), ch.size() * sizeof(float), cudaMemcpyHostToDevice));
            plan->chunks.ensure(chunks.size() * sizeof(nbx::ChunkF32));
            NBX_CUDA(cudaMemcpy(plan->chunks.p, chunks.data(), chunks.size() * sizeof(nbx::ChunkF32),
                                cudaMemcpyHostToDevice));
            P.chunks = static_cast<const nbx::ChunkF32*>(plan->chunks.p);
            P.n_chunks = (int32_t)chunks.size();
            if (!table_current && !plan->hash) {
                plan->table.ensure(cells_alloc * sizeof(float));
                NBX_CUDA(cudaMemcpy(plan->table.p, plan->host_table.p, cells_alloc * sizeof(float),
                                    cudaMemcpyHostToDevice));
            }
        } else {
            // Channel-recurrence variant (sincg): channels sorted by 1/lambda and cut into
            // runs whose 1/lambda are an arithmetic progression to within 1e-14 of phase
            // (|S (iv_k - iv_0 - k delta)| <= 1e-14 for every reachable S); used when the
            // runs are long enough to amortise their per-run anchors.
            std::vector<int> order(n_src);
            std::vector<double> iv(n_src);
            for (int i = 0; i < n_src; ++i) {
                order[i] = i;
                iv[i] = 1.0 / d->wavelengths[sb + i];  // kernels.py:257
            }
            std::vector<nbx::RunF64> runs;
            const char* rev = std::getenv("NBX_FP64_REC");
            if (d->shape == NBX_SHAPE_SINCG && !(rev && std::atoi(rev) == 0) && n_src >= 2) {
                std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return iv[x] < iv[y]; });
                int b = 0;
                while (b < n_src) {
                    int e = std::min(n_src, b + 128);
                    for (;;) {
                        const int len = e - b;
                        double delta = len > 1 ? (iv[order[e - 1]] - iv[order[b]]) / (double)(len - 1) : 0.0;
                        double dev = 0.0;
                        for (int k = 0; k < len; ++k)
                            dev = std::max(dev, std::fabs(iv[order[b + k]] - iv[order[b]] - (double)k * delta));
                        // segmented variant: at most one index change per axis per run
                        const bool span_ok = len == 1 || smax * std::fabs(delta) * (double)(len - 1) <= 0.9;
                        if (len == 1 || (dev * smax <= 1e-14 && span_ok)) {
                            runs.push_back(nbx::RunF64{iv[order[b]], delta, b, e});
                            break;
                        }
                        e = b + len / 2;
                    }
                    b = e;
                }
                if ((int64_t)runs.size() * 8 > n_src) {  // mean run shorter than 8: direct kernel
                    runs.clear();
                    for (int i = 0; i < n_src; ++i) order[i] = i;
                }
            }
            std::vector<double> ch(2 * (size_t)n_src);
            for (int i = 0; i < n_src; ++i) {
                ch[2 * i + 0] = iv[order[i]];
                ch[2 * i + 1] = d->weights[sb + order[i]];
            }
            plan->chan.ensure(ch.size() * sizeof(double));
            NBX_CUDA(cudaMemcpy(plan->chan.p, ch.data(), ch.size() * sizeof(double), cudaMemcpyHostToDevice));
            if (!runs.empty()) {
                // 6: segmented recurrence (default); NBX_FP64_REC=1: the per-channel bracket variant.
                // (Variant 6's shared memory -- channels, runs, per-thread event records -- fits a
                // block up to kMaxShardSources in runs of 8; the check keeps that true.)
                int dev = 0, smem_max = 0;
                NBX_CUDA(cudaGetDevice(&dev));
                NBX_CUDA(cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
                const bool seg_fits = nbx::seg_f64_smem_bytes(n_src, (int)runs.size()) <= (size_t)smem_max;
                plan->kernel_variant = (rev && std::atoi(rev) == 1) || !seg_fits ? 4 : 6;
                plan->runs.ensure(runs.size() * sizeof(nbx::RunF64));
                NBX_CUDA(cudaMemcpy(plan->runs.p, runs.data(), runs.size() * sizeof(nbx::RunF64),
                                    cudaMemcpyHostToDevice));
                P.runs = static_cast<const nbx::RunF64*>(plan->runs.p);
                P.n_runs = (int32_t)runs.size();
            }
            if (!table_current && !plan->hash) {
                plan->table.ensure(cells * sizeof(double));
                NBX_CUDA(cudaMemcpy(plan->table.p, plan->host_table.p, cells * sizeof(double),
                                    cudaMemcpyHostToDevice));
            }
        }
        if (!table_current && !plan->hash) {
            tk.compute = compute;
            tk.default_f = d->default_f;
            tk.sH = P.sH;
            tk.sK = P.sK;
            for (int a = 0; a < 3; ++a) tk.hmax[a] = hmax[a];
            tk.sigma = sigma;
            tk.maxf2 = maxf2;
            tk.dev = plan->table.p;
            tk.hkl.assign(d->hkl, d->hkl + 3 * (size_t)d->n_entries);
            tk.amp.assign(d->amplitudes, d->amplitudes + d->n_entries);
            tk.valid = true;
        }
        pt.mark("channels+upload");
        if (n_src > kMaxShardSources)
            throw ArgError("too many sources in one plan (max " + std::to_string(kMaxShardSources) +
                           "; nbx_spots splits longer spectra, or shard with src_begin/src_end)");

        plan->bases.ensure(sizeof(double) * 9 * d->n_domains);
        NBX_CUDA(cudaMemcpy(plan->bases.p, d->bases, sizeof(double) * 9 * d->n_domains, cudaMemcpyHostToDevice));
        plan->panels.ensure(sizeof(nbx::DevPanel) * hp.size());
        NBX_CUDA(cudaMemcpy(plan->panels.p, hp.data(), sizeof(nbx::DevPanel) * hp.size(), cudaMemcpyHostToDevice));

        // kernel parameter block
        P.panels = static_cast<const nbx::DevPanel*>(plan->panels.p);
        P.n_panels = d->n_panels;
        P.oversample = os;
        P.bases = static_cast<const double*>(plan->bases.p);
        P.n_dom = d->n_domains;
        P.n_src = n_chan_entries;
        P.chan = plan->chan.p;
        for (int a = 0; a < 3; ++a) {
            P.beam[a] = d->beam_direction[a];
            P.n_cells_d[a] = (double)d->n_cells[a];
            P.n_cells_f[a] = (float)d->n_cells[a];
            P.n_pi_f[a] = (float)(3.14159265358979323846 * (double)d->n_cells[a]);
        }
        P.nnn_d = (double)d->n_cells[0] * d->n_cells[1] * d->n_cells[2];
        P.nnn_f = (float)P.nnn_d;
        P.pol_on = d->polarization_on ? 1 : 0;
        P.table = plan->table.p;
        if (compute == NBX_COMPUTE_FP32 && !plan->hash && !plan->wide) {
            // texture view of the power-of-two table for the packed loop's gathers
            const size_t tb = (size_t)cells_alloc * sizeof(float);
            if (!plan->tex || plan->tex_ptr != plan->table.p || plan->tex_bytes != tb) {
                plan->release_tex();
                cudaResourceDesc rd{};
                rd.resType = cudaResourceTypeLinear;
                rd.res.linear.devPtr = plan->table.p;
                rd.res.linear.desc = cudaCreateChannelDesc<float>();
                rd.res.linear.sizeInBytes = tb;
                cudaTextureDesc td{};
                td.readMode = cudaReadModeElementType;
                NBX_CUDA(cudaCreateTextureObject(&plan->tex, &rd, &td, nullptr));
                plan->tex_ptr = plan->table.p;
                plan->tex_bytes = tb;
            }
            P.table_tex = plan->tex;
        }
        P.max_slow = max_slow;
        P.max_fast = max_fast;
        P.out_scale = plan->out_scale;
        P.raw_scale = 1.0 / sigma;
        setup_background(d, P, plan->bg);

        pt.mark("rest");
        nbx_plan_info_t& I = plan->info;
        I.n_pixels = plan->n_pixels;
        I.steps = plan->steps;
        if (!plan->hash) I.table_cells = cells_alloc;  // hash: build_hash recorded the slot count
        for (int a = 0; a < 3; ++a) {
            I.table_lo[a] = P.lo[a];
            I.table_dim[a] = (int32_t)dims[a];
        }
        I.compute = compute;
        I.table_kind = plan->hash ? 2 : (plan->wide ? 1 : 0);
        I.channel_runs = P.n_runs;
        I.kernel_variant = plan->kernel_variant;
        I.scale = plan->scale;
        return plan;
    } catch (...) {
        if (!reuse) delete plan;
        throw;
    }
}

size_t out_elem_bytes(int mode) {
    return (mode == NBX_OUT_F32 || mode == NBX_OUT_IMAGE_F32) ? 4 : 8;  // F64 / ADD / RAW / IMAGE_F64: f64
}

void check_mode(int mode) {
    if (mode < NBX_OUT_F32 || mode > NBX_OUT_RAW_STORE_F64) throw ArgError("unknown output mode");
}

// Three fault slots per launch: spots, background, f32 downcast of the image.
constexpr int kFaultSlots = 3;

int64_t pick_fault(Ctx* ctx, const unsigned long long* fault) {
    for (int s = 0; s < kFaultSlots; ++s) {
        if (fault[s] != ~0ull) {
            ctx->fault_stage = s;
            return (int64_t)fault[s];
        }
    }
    return -1;
}

// Launch the spot kernel of `plan` over rows [row0, row1) of every panel.
void launch_rows(Plan* plan, int mode, void* dout, unsigned long long* fault, cudaStream_t st, int row0, int row1) {
    nbx::SpotsParams P = plan->P;
    P.out_mode = mode;
    P.out = dout;
    P.fault = fault;
    P.fault_bg = fault + 1;  // fault_bg[1] = the downcast slot
    P.row0 = row0;
    P.max_slow = row1;
    NBX_CUDA(nbx::launch_spots(P, plan->kernel_variant, plan->shape, plan->hash ? 2 : (plan->wide ? 1 : 0), st));
}

// Enqueue one spot launch of `plan` into device buffer `dout` with fault slots `fault`.
void enqueue_plan(Plan* plan, int mode, void* dout, unsigned long long* fault, cudaStream_t st) {
    NBX_CUDA(cudaMemsetAsync(fault, 0xFF, kFaultSlots * sizeof(unsigned long long), st));
    launch_rows(plan, mode, dout, fault, st, 0, plan->P.max_slow);
}

// Row bands of a pipelined host-output run (0: one launch, copy afterwards).
constexpr int kBands = 8;
int band_rows(const Plan* plan, int mode, int on_device) {
    const bool write_only = mode == NBX_OUT_F32 || mode == NBX_OUT_F64 || mode == NBX_OUT_IMAGE_F32 ||
                            mode == NBX_OUT_IMAGE_F64;
    if (on_device || !write_only || !plan->uniform_panels || plan->n_pixels < (int64_t(1) << 20)) return 0;
    const char* ev = std::getenv("NBX_BANDS");
    const int nb = ev ? std::max(1, std::min(16, std::atoi(ev))) : kBands;
    if (nb <= 1) return 0;
    const int rows = plan->P.max_slow;
    return ((rows + nb - 1) / nb + 7) / 8 * 8;  // whole 8-row block lines per band
}

void ensure_band_resources(Ctx* ctx) {
    if (!ctx->stream2) NBX_CUDA(cudaStreamCreateWithFlags(&ctx->stream2, cudaStreamNonBlocking));
    if (!ctx->copy_stream) NBX_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    if (!ctx->join_ev) NBX_CUDA(cudaEventCreateWithFlags(&ctx->join_ev, cudaEventDisableTiming));
    for (auto& e : ctx->band_ev)
        if (!e) NBX_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
}

// Run a plan into `out`; returns the lowest non-finite pixel or -1.
//
// With a host `out` the image is computed in row bands that alternate between
// two compute streams, and band b's download (a 2-D copy: the same rows of every
// panel) runs on the copy stream while later bands compute, so only the last
// band's download is exposed (the reference-facing call's end-to-end time).
int64_t run_plan(Plan* plan, int mode, void* out, int on_device) {
    NvtxRange nvtx(on_device ? "nbx spots (device output)" : "nbx spots (launch + download)");
    check_mode(mode);
    if (!out) throw ArgError("output buffer is NULL");
    Ctx* ctx = plan->ctx;
    NBX_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    const size_t es = out_elem_bytes(mode);
    const size_t bytes = (size_t)plan->n_pixels * es;
    void* dout = out;
    if (!on_device) {
        ctx->out_scratch.ensure(bytes);
        dout = ctx->out_scratch.p;
        if (mode == NBX_OUT_ADD_F64 || mode == NBX_OUT_RAW_F64)
            NBX_CUDA(cudaMemcpyAsync(dout, out, bytes, cudaMemcpyHostToDevice, st));
    }
    ctx->fault.ensure(kFaultSlots * sizeof(unsigned long long));
    unsigned long long* dfault = static_cast<unsigned long long*>(ctx->fault.p);
    unsigned long long fault[kFaultSlots] = {~0ull, ~0ull, ~0ull};
    const int per = band_rows(plan, mode, on_device);
    if (per == 0) {
        NBX_CUDA(cudaEventRecord(ctx->ev0, st));
        enqueue_plan(plan, mode, dout, dfault, st);
        NBX_CUDA(cudaEventRecord(ctx->ev1, st));
        NBX_CUDA(cudaMemcpyAsync(fault, dfault, sizeof(fault), cudaMemcpyDeviceToHost, st));
        if (!on_device) NBX_CUDA(cudaMemcpyAsync(out, dout, bytes, cudaMemcpyDeviceToHost, st));
        NBX_CUDA(cudaStreamSynchronize(st));
    } else {
        ensure_band_resources(ctx);
        cudaStream_t s2 = ctx->stream2, cs = ctx->copy_stream;
        const int rows = plan->P.max_slow, fast = plan->P.max_fast;
        const size_t pitch = (size_t)rows * fast * es;  // one panel
        NBX_CUDA(cudaEventRecord(ctx->ev0, st));
        NBX_CUDA(cudaMemsetAsync(dfault, 0xFF, kFaultSlots * sizeof(unsigned long long), st));
        NBX_CUDA(cudaEventRecord(ctx->join_ev, st));
        NBX_CUDA(cudaStreamWaitEvent(s2, ctx->join_ev, 0));
        int nb = 0;
        for (int r0 = 0; r0 < rows; r0 += per, ++nb) {  // all launches first: the copies below block the host
            cudaStream_t s = (nb & 1) ? s2 : st;
            launch_rows(plan, mode, dout, dfault, s, r0, std::min(rows, r0 + per));
            NBX_CUDA(cudaEventRecord(ctx->band_ev[nb], s));
        }
        NBX_CUDA(cudaEventRecord(ctx->join_ev, s2));
        NBX_CUDA(cudaStreamWaitEvent(st, ctx->join_ev, 0));
        NBX_CUDA(cudaEventRecord(ctx->ev1, st));
        for (int b = 0; b < nb; ++b) {
            const int r0 = b * per, r1 = std::min(rows, r0 + per);
            const size_t off = (size_t)r0 * fast * es, width = (size_t)(r1 - r0) * fast * es;
            NBX_CUDA(cudaStreamWaitEvent(cs, ctx->band_ev[b], 0));
            NBX_CUDA(cudaMemcpy2DAsync(static_cast<char*>(out) + off, pitch, static_cast<const char*>(dout) + off,
                                       pitch, width, (size_t)plan->P.n_panels, cudaMemcpyDeviceToHost, cs));
        }
        NBX_CUDA(cudaMemcpyAsync(fault, dfault, sizeof(fault), cudaMemcpyDeviceToHost, st));
        NBX_CUDA(cudaStreamSynchronize(cs));
        NBX_CUDA(cudaStreamSynchronize(st));
    }
    plan->timed = true;
    NBX_CUDA(cudaEventElapsedTime(&plan->last_ms, ctx->ev0, ctx->ev1));
    return pick_fault(ctx, fault);
}

// zlib's CRC-32 (reflected 0xEDB88320), slicing-by-8.
struct Crc32Tables {
    uint32_t t[8][256];
    Crc32Tables() {
        for (uint32_t i = 0; i < 256; ++i) {
            uint32_t c = i;
            for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
            t[0][i] = c;
        }
        for (uint32_t i = 0; i < 256; ++i)
            for (int s = 1; s < 8; ++s) t[s][i] = (t[s - 1][i] >> 8) ^ t[0][t[s - 1][i] & 0xFF];
    }
};

uint32_t crc32_update(uint32_t crc, const unsigned char* p, size_t n) {
    static const Crc32Tables T;
    uint32_t c = ~crc;
    while (n >= 8) {
        uint32_t lo, hi;
        std::memcpy(&lo, p, 4);
        std::memcpy(&hi, p + 4, 4);
        lo ^= c;
        c = T.t[7][lo & 0xFF] ^ T.t[6][(lo >> 8) & 0xFF] ^ T.t[5][(lo >> 16) & 0xFF] ^ T.t[4][lo >> 24] ^
            T.t[3][hi & 0xFF] ^ T.t[2][(hi >> 8) & 0xFF] ^ T.t[1][(hi >> 16) & 0xFF] ^ T.t[0][hi >> 24];
        p += 8;
        n -= 8;
    }
    while (n--) c = T.t[0][(c ^ *p++) & 0xFF] ^ (c >> 8);
    return ~c;
}

thread_local std::string g_noctx_err;

void set_err(void* ctxp, const std::string& msg) {
    if (ctxp)
        static_cast<Ctx*>(ctxp)->err = msg;
    else
        g_noctx_err = msg;
}

template <typename F>
int guarded(void* ctxp, F&& f) {
    try {
        return f();
    } catch (const ArgError& e) {
        set_err(ctxp, e.what());
        return NBX_ERR_ARG;
    } catch (const CudaError& e) {
        set_err(ctxp, e.what());
        return NBX_ERR_CUDA;
    } catch (const std::bad_alloc&) {
        set_err(ctxp, "host allocation failed");
        return NBX_ERR_ARG;
    } catch (const std::exception& e) {
        set_err(ctxp, e.what());
        return NBX_ERR_CUDA;
    }
}

int fault_status(void* ctxp, int64_t bad, int64_t* first_bad) {
    if (first_bad) *first_bad = bad;
    if (bad >= 0) {
        set_err(ctxp, "non-finite value at pixel " + std::to_string(bad));
        return NBX_ERR_NUMERICAL;
    }
    return NBX_OK;
}

}  // namespace

extern "C" {

int nbx_version(void) { return NBX_VERSION; }

int64_t nbx_struct_size(int which) {
    switch (which) {
        case 0: return (int64_t)sizeof(nbx_panel);
        case 1: return (int64_t)sizeof(nbx_spots_desc);
        case 2: return (int64_t)sizeof(nbx_plan_info_t);
        default: return 0;
    }
}

int nbx_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

void* nbx_ctx_create(int device) {
    try {
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || n <= 0) {
            cudaGetLastError();
            g_noctx_err = "no CUDA device available";
            return nullptr;
        }
        if (device < 0 || device >= n) {
            g_noctx_err = "device index out of range";
            return nullptr;
        }
        auto ctx = new Ctx();
        ctx->device = device;
        if (cudaSetDevice(device) != cudaSuccess || cudaStreamCreateWithFlags(&ctx->own, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreate(&ctx->ev0) != cudaSuccess || cudaEventCreate(&ctx->ev1) != cudaSuccess) {
            g_noctx_err = std::string("CUDA init failed: ") + cudaGetErrorString(cudaGetLastError());
            delete ctx;
            return nullptr;
        }
        ctx->stream = ctx->own;
        return ctx;
    } catch (...) {
        g_noctx_err = "context allocation failed";
        return nullptr;
    }
}

void nbx_ctx_destroy(void* ctxp) {
    if (!ctxp) return;
    Ctx* ctx = static_cast<Ctx*>(ctxp);
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    delete ctx->oneshot;
    ctx->oneshot = nullptr;
    for (int b = 0; b < 2; ++b) {
        delete ctx->camp_plan[b];
        ctx->camp_out[b].release();
        ctx->camp_fault[b].release();
        if (ctx->camp_host[b]) cudaFreeHost(ctx->camp_host[b]);
    }
    if (ctx->camp_fault_host) cudaFreeHost(ctx->camp_fault_host);
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    if (ctx->stream2) cudaStreamDestroy(ctx->stream2);
    if (ctx->join_ev) cudaEventDestroy(ctx->join_ev);
    for (auto e : ctx->band_ev)
        if (e) cudaEventDestroy(e);
    ctx->out_scratch.release();
    ctx->stage_in.release();
    ctx->stats_parts.release();
    ctx->stats_res.release();
    ctx->hist_counts.release();
    ctx->raw_scratch.release();
    ctx->fault.release();
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    if (ctx->own) cudaStreamDestroy(ctx->own);
    delete ctx;
}

const char* nbx_last_error(void* ctxp) {
    if (!ctxp) return g_noctx_err.c_str();
    return static_cast<Ctx*>(ctxp)->err.c_str();
}

int nbx_ctx_set_stream(void* ctxp, void* stream) {
    if (!ctxp) return NBX_ERR_ARG;
    Ctx* ctx = static_cast<Ctx*>(ctxp);
    ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own;
    return NBX_OK;
}

int nbx_ctx_synchronize(void* ctxp) {
    return guarded(ctxp, [&] {
        if (!ctxp) throw ArgError("NULL context");
        Ctx* ctx = static_cast<Ctx*>(ctxp);
        NBX_CUDA(cudaSetDevice(ctx->device));
        NBX_CUDA(cudaStreamSynchronize(ctx->stream));
        return NBX_OK;
    });
}

int64_t nbx_output_pixels(const nbx_spots_desc* d) {
    try {
        return count_pixels(d);
    } catch (...) {
        return -1;
    }
}

void* nbx_plan_create(void* ctxp, const nbx_spots_desc* d, int compute) {
    Plan* plan = nullptr;
    int st = guarded(ctxp, [&] {
        if (!ctxp) throw ArgError("NULL context");
        NBX_CUDA(cudaSetDevice(static_cast<Ctx*>(ctxp)->device));
        plan = build_plan(static_cast<Ctx*>(ctxp), d, compute);
        return NBX_OK;
    });
    return st == NBX_OK ? plan : nullptr;
}

int nbx_plan_run(void* planp, int out_mode, void* out, int out_on_device, int64_t* first_bad) {
    if (!planp) return NBX_ERR_ARG;
    Plan* plan = static_cast<Plan*>(planp);
    int64_t bad = -1;
    int st = guarded(plan->ctx, [&] {
        bad = run_plan(plan, out_mode, out, out_on_device);
        return NBX_OK;
    });
    if (st != NBX_OK) return st;
    return fault_status(plan->ctx, bad, first_bad);
}

int nbx_plan_info(void* planp, nbx_plan_info_t* info) {
    if (!planp || !info) return NBX_ERR_ARG;
    *info = static_cast<Plan*>(planp)->info;
    return NBX_OK;
}

double nbx_plan_last_kernel_ms(void* planp) {
    if (!planp) return -1.0;
    return static_cast<Plan*>(planp)->last_ms;
}

void nbx_plan_destroy(void* planp) {
    if (!planp) return;
    Plan* plan = static_cast<Plan*>(planp);
    cudaSetDevice(plan->ctx->device);
    cudaStreamSynchronize(plan->ctx->stream);
    delete plan;
}

int nbx_finalize(void* ctxp, const double* raw, int64_t n, double scale, int out_mode, void* out, int out_on_device,
                 int64_t* first_bad);


int nbx_spots(void* ctxp, const nbx_spots_desc* d, int compute, int out_mode, void* out, int out_on_device,
              int64_t* first_bad) {
    int64_t bad = -1;
    if (ctxp && d && d->n_sources > 0) {
        const int sb = d->src_begin, se = d->src_end <= 0 ? d->n_sources : d->src_end;
        if (se - sb > kMaxShardSources) {
            // Long spectrum (the reference has no limit): channel shards accumulated as FP64
            // partials with the GLOBAL normalisation, then one scale + store -- exactly a
            // channel-sharded image on one device.  A RAW request receives
            // the shards' partials added into the caller's buffer; an IMAGE request gets the
            // simulate_image accumulator composed stage by stage (below).
            int64_t npix = 0;
            double scale = 0.0;
            const int st = guarded(ctxp, [&] {
                Ctx* ctx = static_cast<Ctx*>(ctxp);
                NBX_CUDA(cudaSetDevice(ctx->device));
                check_mode(out_mode);
                validate(d);
                npix = count_pixels(d);
                nbx_spots_desc sh = *d;
                if (!(sh.norm > 0)) {  // kernels.py:243-245 over the WHOLE spectrum
                    double wsum = 0.0;
                    for (int i = 0; i < d->n_sources; ++i) wsum += d->weights[i];
                    sh.norm = wsum * (double)d->n_domains * (double)(d->oversample * d->oversample);
                }
                const bool raw_out = out_mode == NBX_OUT_RAW_F64 || out_mode == NBX_OUT_RAW_STORE_F64;
                void* acc = out;
                int acc_on_device = out_on_device;
                if (out_mode == NBX_OUT_RAW_STORE_F64) {  // store semantics: start from zero
                    if (out_on_device)
                        NBX_CUDA(cudaMemsetAsync(out, 0, (size_t)npix * sizeof(double), ctx->stream));
                    else
                        std::memset(out, 0, (size_t)npix * sizeof(double));
                }
                if (!raw_out) {
                    ctx->raw_scratch.ensure((size_t)npix * sizeof(double));
                    NBX_CUDA(cudaMemsetAsync(ctx->raw_scratch.p, 0, (size_t)npix * sizeof(double), ctx->stream));
                    acc = ctx->raw_scratch.p;
                    acc_on_device = 1;
                }
                if (!ctx->oneshot) ctx->oneshot = new Plan();
                for (int s0 = sb; s0 < se; s0 += kMaxShardSources) {
                    sh.src_begin = s0;
                    sh.src_end = std::min(se, s0 + kMaxShardSources);
                    Plan* plan = build_plan(ctx, &sh, compute, ctx->oneshot);
                    scale = plan->scale;
                    run_plan(plan, NBX_OUT_RAW_F64, acc, acc_on_device);  // += this shard's partial
                }
                return NBX_OK;
            });
            if (st != NBX_OK || out_mode == NBX_OUT_RAW_F64 || out_mode == NBX_OUT_RAW_STORE_F64) return st;
            Ctx* ctx = static_cast<Ctx*>(ctxp);
            const double* raw = static_cast<const double*>(ctx->raw_scratch.p);
            if (out_mode != NBX_OUT_IMAGE_F64 && out_mode != NBX_OUT_IMAGE_F32)
                return nbx_finalize(ctxp, raw, npix, scale, out_mode, out, out_on_device, first_bad);
            // simulate_image's accumulator, the fused epilogue's stages one after another with
            // the same arithmetic and fault precedence: f64(f32(spots)) (+ f64(f32(background)))
            // (scheduler.py:156-183), then the f32 payload for IMAGE_F32 (io.py:403-434)
            const bool direct = out_mode == NBX_OUT_IMAGE_F64 && out_on_device;
            void* img = out;
            int st2 = guarded(ctxp, [&] {
                if (!direct) {
                    ctx->img_scratch.ensure((size_t)npix * sizeof(double));
                    img = ctx->img_scratch.p;
                }
                NBX_CUDA(cudaMemsetAsync(img, 0, (size_t)npix * sizeof(double), ctx->stream));
                return NBX_OK;
            });
            if (st2 != NBX_OK) return st2;
            ctx->fault_stage = 0;
            st2 = nbx_finalize(ctxp, raw, npix, scale, NBX_OUT_ADD_F64, img, 1, first_bad);
            if (st2 != NBX_OK) return st2;
            if (d->bg_points > 0) {
                st2 = nbx_background(ctxp, d, NBX_OUT_ADD_F64, img, 1, first_bad);  // sets fault_stage 1
                if (st2 != NBX_OK) return st2;
            }
            if (out_mode == NBX_OUT_IMAGE_F64) {
                if (direct) return NBX_OK;
                return guarded(ctxp, [&] {
                    NBX_CUDA(cudaMemcpy(out, img, (size_t)npix * sizeof(double),
                                        out_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost));
                    return NBX_OK;
                });
            }
            st2 = nbx_finalize(ctxp, static_cast<const double*>(img), npix, 1.0, NBX_OUT_F32, out, out_on_device,
                               first_bad);
            if (st2 == NBX_ERR_NUMERICAL) ctx->fault_stage = 2;
            return st2;
        }
    }
    int st = guarded(ctxp, [&] {
        if (!ctxp) throw ArgError("NULL context");
        NBX_CUDA(cudaSetDevice(static_cast<Ctx*>(ctxp)->device));
        check_mode(out_mode);
        Ctx* ctx = static_cast<Ctx*>(ctxp);
        const auto t0 = std::chrono::steady_clock::now();
        if (!ctx->oneshot) ctx->oneshot = new Plan();
        Plan* plan = build_plan(ctx, d, compute, ctx->oneshot);
        const auto t1 = std::chrono::steady_clock::now();
        bad = run_plan(plan, out_mode, out, out_on_device);
        const auto t2 = std::chrono::steady_clock::now();
        const float kms = plan->last_ms;
        if (trace_enabled()) {
            const auto t3 = std::chrono::steady_clock::now();
            auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
            std::fprintf(stderr, "[nbx] spots: plan %.2f ms, run %.2f ms (kernel %.2f ms), release %.2f ms\n",
                         ms(t0, t1), ms(t1, t2), kms, ms(t2, t3));
        }
        return NBX_OK;
    });
    if (st != NBX_OK) return st;
    return fault_status(ctxp, bad, first_bad);
}

// Device copy of a host input (or the device pointer itself).
const void* stage_input(Ctx* ctx, DevBuf& tmp, const void* data, size_t bytes, int on_device, cudaStream_t s) {
    if (on_device) return data;
    tmp.ensure(bytes);
    NBX_CUDA(cudaMemcpyAsync(tmp.p, data, bytes, cudaMemcpyHostToDevice, s));
    (void)ctx;
    return tmp.p;
}

int nbx_image_stats(void* ctxp, const void* data, int64_t n, int dtype, int on_device, double* out4) {
    return guarded(ctxp, [&] {
        if (!ctxp || !out4 || !data) throw ArgError("invalid image_stats arguments");
        if (n < 1) throw ArgError("image_stats requires a non-empty buffer");
        if (dtype != 0 && dtype != 1) throw ArgError("dtype must be 0 (f32) or 1 (f64)");
        Ctx* ctx = static_cast<Ctx*>(ctxp);
        NBX_CUDA(cudaSetDevice(ctx->device));
        cudaStream_t s = ctx->stream;
        DevBuf& in = ctx->stage_in;
        DevBuf& parts = ctx->stats_parts;
        DevBuf& res = ctx->stats_res;
        const void* d = stage_input(ctx, in, data, (size_t)n * (dtype ? 8 : 4), on_device, s);
        parts.ensure(nbx::stats_scratch_bytes(n));
        res.ensure(3 * sizeof(double));
        NBX_CUDA(nbx::launch_stats(d, n, dtype, parts.p, static_cast<double*>(res.p), s));
        double h[3];
        NBX_CUDA(cudaMemcpyAsync(h, res.p, sizeof(h), cudaMemcpyDeviceToHost, s));
        NBX_CUDA(cudaStreamSynchronize(s));
        out4[0] = h[0];
        out4[1] = h[1];
        out4[2] = h[2] / (double)n;
        out4[3] = h[2];
        return NBX_OK;
    });
}

int nbx_image_histogram(void* ctxp, const void* data, int64_t n, int dtype, int on_device, int n_bins, double lo,
                        double hi, int64_t* counts, int64_t* underflow, int64_t* overflow) {
    return guarded(ctxp, [&] {
        if (!ctxp || !data || !counts) throw ArgError("invalid image_histogram arguments");
        if (!(lo < hi)) throw ArgError("histogram range must satisfy lo < hi");
        if (n_bins < 1) throw ArgError("n_bins must be >= 1");
        if (n < 1) throw ArgError("image_histogram requires a non-empty buffer");
        if (dtype != 0 && dtype != 1) throw ArgError("dtype must be 0 (f32) or 1 (f64)");
        Ctx* ctx = static_cast<Ctx*>(ctxp);
        NBX_CUDA(cudaSetDevice(ctx->device));
        cudaStream_t s = ctx->stream;
        DevBuf& in = ctx->stage_in;
        DevBuf& cnt = ctx->hist_counts;
        const void* d = stage_input(ctx, in, data, (size_t)n * (dtype ? 8 : 4), on_device, s);
        cnt.ensure(sizeof(unsigned long long) * ((size_t)n_bins + 2));
        NBX_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long) * ((size_t)n_bins + 2), s));
        NBX_CUDA(nbx::launch_histogram(d, n, dtype, n_bins, lo, hi, static_cast<unsigned long long*>(cnt.p), s));
        std::vector<unsigned long long> h((size_t)n_bins + 2);
        NBX_CUDA(cudaMemcpyAsync(h.data(), cnt.p, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
        NBX_CUDA(cudaStreamSynchronize(s));
        for (int b = 0; b < n_bins; ++b) counts[b] = (int64_t)h[b + 1];
        if (underflow) *underflow = (int64_t)h[0];
        if (overflow) *overflow = (int64_t)h[(size_t)n_bins + 1];
        return NBX_OK;
    });
}

uint32_t nbx_crc32(uint32_t crc, const void* data, int64_t n) {
    if (!data || n <= 0) return crc;
    return crc32_update(crc, static_cast<const unsigned char*>(data), (size_t)n);
}

int nbx_campaign(void* ctxp, const nbx_spots_desc* descs, int n_images, int compute, const char* const* paths,
                 uint32_t* crcs, int64_t* image_fault) {
    constexpr int64_t kNotRun = -2, kIoFailed = -3;
    int stop = NBX_OK;  // NBX_ERR_NUMERICAL (non-finite payload) or NBX_ERR_IO end the campaign early
    std::string stop_msg;
    if (image_fault)
        for (int i = 0; i < n_images; ++i) image_fault[i] = kNotRun;
    int st = guarded(ctxp, [&]() -> int {
        if (!ctxp) throw ArgError("NULL context");
        if (n_images < 0 || (n_images > 0 && (!descs || !paths || !crcs || !image_fault)))
            throw ArgError("invalid campaign arguments");
        Ctx* ctx = static_cast<Ctx*>(ctxp);
        NBX_CUDA(cudaSetDevice(ctx->device));
        if (!ctx->copy_stream) NBX_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
        cudaStream_t cs = ctx->stream, ds = ctx->copy_stream;
        cudaEvent_t kdone[2], copied[2];
        for (int b = 0; b < 2; ++b) {
            NBX_CUDA(cudaEventCreateWithFlags(&kdone[b], cudaEventDisableTiming));
            NBX_CUDA(cudaEventCreateWithFlags(&copied[b], cudaEventDisableTiming));
            if (!ctx->camp_plan[b]) ctx->camp_plan[b] = new Plan();
            ctx->camp_fault[b].ensure(kFaultSlots * sizeof(unsigned long long));
        }
        struct Events {
            cudaEvent_t* e;
            ~Events() {
                for (int i = 0; i < 4; ++i) cudaEventDestroy(e[i]);
            }
        };
        cudaEvent_t all[4] = {kdone[0], kdone[1], copied[0], copied[1]};
        Events guard{all};
        // fault slots come back through PINNED memory: a cudaMemcpyAsync into pageable memory
        // would block the host until the copy stream reached it (i.e. until the NEXT image's
        // kernel finished), serialising the write-out with the GPU
        if (!ctx->camp_fault_host)
            NBX_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ctx->camp_fault_host),
                                   2 * kFaultSlots * sizeof(unsigned long long), cudaHostAllocDefault));
        unsigned long long* hfault[2] = {ctx->camp_fault_host, ctx->camp_fault_host + kFaultSlots};
        size_t bytes[2] = {0, 0};
        // render image i into slot i % 2: plan build (host), launch, then async D2H + fault read
        auto launch = [&](int i) {
            NvtxRange nvtx("nbx campaign launch");
            const int b = i & 1;
            Plan* plan = build_plan(ctx, descs + i, compute, ctx->camp_plan[b]);
            bytes[b] = (size_t)plan->n_pixels * 4;
            ctx->camp_out[b].ensure(bytes[b]);
            enqueue_plan(plan, NBX_OUT_IMAGE_F32, ctx->camp_out[b].p,
                         static_cast<unsigned long long*>(ctx->camp_fault[b].p), cs);
            NBX_CUDA(cudaEventRecord(kdone[b], cs));
            NBX_CUDA(cudaStreamWaitEvent(ds, kdone[b], 0));
            NBX_CUDA(cudaMemcpyAsync(hfault[b], ctx->camp_fault[b].p, kFaultSlots * sizeof(unsigned long long),
                                     cudaMemcpyDeviceToHost, ds));
            NBX_CUDA(cudaMemcpyAsync(ctx->camp_host[b], ctx->camp_out[b].p, bytes[b], cudaMemcpyDeviceToHost, ds));
            NBX_CUDA(cudaEventRecord(copied[b], ds));
        };
        // pinned staging sized once for the largest image (never reallocated mid-pipeline)
        size_t max_bytes = 0;
        for (int i = 0; i < n_images; ++i) max_bytes = std::max(max_bytes, (size_t)count_pixels(descs + i) * 4);
        if (ctx->camp_host_bytes < max_bytes) {
            for (int q = 0; q < 2; ++q) {
                if (ctx->camp_host[q]) cudaFreeHost(ctx->camp_host[q]);
                ctx->camp_host[q] = nullptr;
            }
            ctx->camp_host_bytes = 0;
            for (int q = 0; q < 2; ++q) NBX_CUDA(cudaMallocHost(&ctx->camp_host[q], max_bytes));
            ctx->camp_host_bytes = max_bytes;
        }
        // false (and the campaign stops) when the file cannot be written
        auto write_image = [&](int i, const void* data, size_t nbytes) -> bool {
            crcs[i] = crc32_update(0, static_cast<const unsigned char*>(data), nbytes);
            FILE* fh = std::fopen(paths[i], "wb");
            bool ok = fh != nullptr;
            if (fh) {
                ok = std::fwrite(data, 1, nbytes, fh) == nbytes;
                ok = (std::fclose(fh) == 0) && ok;
            }
            if (!ok) {
                image_fault[i] = kIoFailed;
                stop = NBX_ERR_IO;
                stop_msg = std::string("cannot write ") + paths[i] + ": " + std::strerror(errno);
                return false;
            }
            image_fault[i] = -1;
            return true;
        };
        // a fault of image i: spots / background stage -> flagged, the campaign continues;
        // a non-finite f32 payload -> the campaign stops (write_image refuses it, io.py:409-411)
        auto fault = [&](int i, int64_t pixel, int stage) -> bool {
            image_fault[i] = ((int64_t)stage << 40) | pixel;
            if (stage == 2) {
                stop = NBX_ERR_NUMERICAL;
                stop_msg = "refusing to write non-finite pixel " + std::to_string(pixel) + " of campaign image " +
                           std::to_string(i);
                return false;
            }
            return true;
        };
        bool any_long = false;  // a spectrum longer than one launch: nbx_spots' sharded image path
        for (int i = 0; i < n_images; ++i) {
            const int sb = descs[i].src_begin, se = descs[i].src_end <= 0 ? descs[i].n_sources : descs[i].src_end;
            any_long |= se - sb > kMaxShardSources;
        }
        if (any_long) {  // image by image, not pipelined (rare: > 8192 sources per image)
            for (int i = 0; i < n_images; ++i) {
                int64_t bad = -1;
                const int s2 = nbx_spots(ctx, descs + i, compute, NBX_OUT_IMAGE_F32, ctx->camp_host[0], 0, &bad);
                if (s2 == NBX_ERR_NUMERICAL) {
                    if (!fault(i, bad, ctx->fault_stage)) return NBX_OK;
                    continue;
                }
                if (s2 != NBX_OK) return s2;
                if (!write_image(i, ctx->camp_host[0], (size_t)count_pixels(descs + i) * 4)) return NBX_OK;
            }
            return NBX_OK;
        }
        if (n_images > 0) launch(0);
        for (int i = 0; i < n_images; ++i) {
            const int b = i & 1;
            if (i + 1 < n_images) launch(i + 1);  // overlaps the write-out of image i below
            NBX_CUDA(cudaEventSynchronize(copied[b]));
            const int64_t bad = pick_fault(ctx, hfault[b]);
            if (bad >= 0) {
                if (fault(i, bad, ctx->fault_stage)) continue;  // flagged: skip the write, keep going
                NBX_CUDA(cudaStreamSynchronize(cs));
                NBX_CUDA(cudaStreamSynchronize(ds));
                return NBX_OK;
            }
            const auto t0 = std::chrono::steady_clock::now();
            NvtxRange nvtx("nbx campaign crc + write");
            if (!write_image(i, ctx->camp_host[b], bytes[b])) {
                NBX_CUDA(cudaStreamSynchronize(cs));
                NBX_CUDA(cudaStreamSynchronize(ds));
                return NBX_OK;
            }
            if (trace_enabled()) {
                const auto t1 = std::chrono::steady_clock::now();
                std::fprintf(stderr, "[nbx] campaign image %d: crc + write %.2f ms\n", i,
                             std::chrono::duration<double, std::milli>(t1 - t0).count());
            }
        }
        return NBX_OK;
    });
    if (st != NBX_OK) return st;
    if (stop != NBX_OK) set_err(ctxp, stop_msg);
    return stop;
}

int nbx_fault_stage(void* ctxp) { return ctxp ? static_cast<Ctx*>(ctxp)->fault_stage : 0; }

int nbx_background(void* ctxp, const nbx_spots_desc* d, int out_mode, void* out, int out_on_device,
                   int64_t* first_bad) {
    int64_t bad = -1;
    int st = guarded(ctxp, [&] {
        if (!ctxp) throw ArgError("NULL context");
        if (out_mode != NBX_OUT_F32 && out_mode != NBX_OUT_F64 && out_mode != NBX_OUT_ADD_F64)
            throw ArgError("background output mode must be F32, F64 or ADD_F64");
        if (!out) throw ArgError("output buffer is NULL");
        count_pixels(d);
        for (int i = 0; i < d->n_panels; ++i) {
            const nbx_panel& p = d->panels[i];
            if (!(p.pixel_size > 0) || !(p.distance > 0)) throw ArgError("invalid panel");
            check_unit(p.fast_axis, "fast_axis");
            check_unit(p.slow_axis, "slow_axis");
        }
        check_unit(d->beam_direction, "beam_direction");
        if (d->n_sources < 1 || !d->wavelengths || !d->weights) throw ArgError("spectrum needs samples");
        if (d->bg_points < 2) throw ArgError("background profile needs at least 2 points");
        Ctx* ctx = static_cast<Ctx*>(ctxp);
        NBX_CUDA(cudaSetDevice(ctx->device));
        cudaStream_t s = ctx->stream;
        if (!ctx->oneshot) ctx->oneshot = new Plan();
        Plan* plan = ctx->oneshot;
        plan->P = nbx::SpotsParams{};
        nbx::SpotsParams& P = plan->P;
        int max_slow = 0, max_fast = 0;
        int64_t npix = 0, subs = 0;
        const std::vector<nbx::DevPanel> hp = make_panels(d, &max_slow, &max_fast, &npix, &subs);
        plan->panels.ensure(sizeof(nbx::DevPanel) * hp.size());
        NBX_CUDA(cudaMemcpy(plan->panels.p, hp.data(), sizeof(nbx::DevPanel) * hp.size(), cudaMemcpyHostToDevice));
        P.panels = static_cast<const nbx::DevPanel*>(plan->panels.p);
        P.n_panels = d->n_panels;
        P.max_slow = max_slow;
        P.max_fast = max_fast;
        for (int a = 0; a < 3; ++a) P.beam[a] = d->beam_direction[a];
        P.pol_on = d->polarization_on ? 1 : 0;
        setup_background(d, P, plan->bg);
        const size_t bytes = (size_t)npix * (out_mode == NBX_OUT_F32 ? 4 : 8);
        void* dout = out;
        if (!out_on_device) {
            ctx->out_scratch.ensure(bytes);
            dout = ctx->out_scratch.p;
            if (out_mode == NBX_OUT_ADD_F64) NBX_CUDA(cudaMemcpyAsync(dout, out, bytes, cudaMemcpyHostToDevice, s));
        }
        ctx->fault.ensure(kFaultSlots * sizeof(unsigned long long));
        NBX_CUDA(cudaMemsetAsync(ctx->fault.p, 0xFF, kFaultSlots * sizeof(unsigned long long), s));
        P.out_mode = out_mode;
        P.out = dout;
        P.fault = static_cast<unsigned long long*>(ctx->fault.p);
        P.fault_bg = P.fault + 1;
        NBX_CUDA(nbx::launch_background(P, s));
        unsigned long long f[2] = {~0ull, ~0ull};
        NBX_CUDA(cudaMemcpyAsync(f, ctx->fault.p, sizeof(f), cudaMemcpyDeviceToHost, s));
        if (!out_on_device) NBX_CUDA(cudaMemcpyAsync(out, dout, bytes, cudaMemcpyDeviceToHost, s));
        NBX_CUDA(cudaStreamSynchronize(s));
        ctx->fault_stage = 1;
        bad = f[1] == ~0ull ? -1 : (int64_t)f[1];
        return NBX_OK;
    });
    if (st != NBX_OK) return st;
    return fault_status(ctxp, bad, first_bad);
}

int nbx_spots_batch(void* ctxp, const nbx_spots_desc* descs, int n_images, int compute, int out_mode,
                    void* const* outs, int out_on_device, int64_t* first_bad) {
    if (first_bad) *first_bad = -1;
    if (n_images < 0 || (n_images > 0 && (!descs || !outs))) {
        set_err(ctxp, "invalid batch arguments");
        return NBX_ERR_ARG;
    }
    for (int i = 0; i < n_images; ++i) {
        int64_t bad = -1;
        const int st = nbx_spots(ctxp, descs + i, compute, out_mode, outs[i], out_on_device, &bad);
        if (st != NBX_OK) {
            // report (image, pixel) as image * 2^40 + pixel so callers can locate it
            if (first_bad && bad >= 0) *first_bad = ((int64_t)i << 40) | bad;
            return st;
        }
    }
    return NBX_OK;
}

int nbx_finalize(void* ctxp, const double* raw, int64_t n, double scale, int out_mode, void* out, int out_on_device,
                 int64_t* first_bad) {
    int64_t bad = -1;
    int st = guarded(ctxp, [&] {
        if (!ctxp) throw ArgError("NULL context");
        if (!raw || !out || n < 0) throw ArgError("invalid finalize arguments");
        if (out_mode != NBX_OUT_F32 && out_mode != NBX_OUT_F64 && out_mode != NBX_OUT_ADD_F64)
            throw ArgError("finalize output mode must be F32, F64 or ADD_F64");
        Ctx* ctx = static_cast<Ctx*>(ctxp);
        NBX_CUDA(cudaSetDevice(ctx->device));
        cudaStream_t s = ctx->stream;
        const size_t bytes = (size_t)n * out_elem_bytes(out_mode);
        void* dout = out;
        if (!out_on_device) {
            ctx->out_scratch.ensure(bytes);
            dout = ctx->out_scratch.p;
            if (out_mode == NBX_OUT_ADD_F64) NBX_CUDA(cudaMemcpyAsync(dout, out, bytes, cudaMemcpyHostToDevice, s));
        }
        ctx->fault.ensure(8);
        NBX_CUDA(cudaMemsetAsync(ctx->fault.p, 0xFF, 8, s));
        NBX_CUDA(nbx::launch_finalize(raw, n, scale, out_mode, dout, static_cast<unsigned long long*>(ctx->fault.p), s));
        unsigned long long f = ~0ull;
        NBX_CUDA(cudaMemcpyAsync(&f, ctx->fault.p, 8, cudaMemcpyDeviceToHost, s));
        if (!out_on_device) NBX_CUDA(cudaMemcpyAsync(out, dout, bytes, cudaMemcpyDeviceToHost, s));
        NBX_CUDA(cudaStreamSynchronize(s));
        bad = f == ~0ull ? -1 : (int64_t)f;
        return NBX_OK;
    });
    if (st != NBX_OK) return st;
    return fault_status(ctxp, bad, first_bad);
}

int nbx_ipc_alloc(void* ctxp, int64_t bytes, void** dev, unsigned char* handle) {
    return guarded(ctxp, [&] {
        if (!ctxp || !dev || !handle || bytes <= 0) throw ArgError("invalid ipc_alloc arguments");
        NBX_CUDA(cudaSetDevice(static_cast<Ctx*>(ctxp)->device));
        NBX_CUDA(cudaMalloc(dev, (size_t)bytes));
        cudaIpcMemHandle_t h;
        NBX_CUDA(cudaIpcGetMemHandle(&h, *dev));
        static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
        std::memcpy(handle, &h, sizeof(h));
        return NBX_OK;
    });
}

int nbx_ipc_free(void* ctxp, void* dev) {
    return guarded(ctxp, [&] {
        if (!ctxp) throw ArgError("NULL context");
        NBX_CUDA(cudaSetDevice(static_cast<Ctx*>(ctxp)->device));
        if (dev) NBX_CUDA(cudaFree(dev));
        return NBX_OK;
    });
}

int nbx_ipc_open(void* ctxp, const unsigned char* handle, void** dev) {
    return guarded(ctxp, [&] {
        if (!ctxp || !handle || !dev) throw ArgError("invalid ipc_open arguments");
        NBX_CUDA(cudaSetDevice(static_cast<Ctx*>(ctxp)->device));
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, sizeof(h));
        NBX_CUDA(cudaIpcOpenMemHandle(dev, h, cudaIpcMemLazyEnablePeerAccess));
        return NBX_OK;
    });
}

int nbx_ipc_close(void* ctxp, void* dev) {
    return guarded(ctxp, [&] {
        if (!ctxp) throw ArgError("NULL context");
        NBX_CUDA(cudaSetDevice(static_cast<Ctx*>(ctxp)->device));
        if (dev) NBX_CUDA(cudaIpcCloseMemHandle(dev));
        return NBX_OK;
    });
}

int nbx_reduce_slots(void* ctxp, const double* slots, int n_slots, int64_t n, double scale, int out_mode, void* out,
                     int out_on_device, int64_t* first_bad) {
    int64_t bad = -1;
    int st = guarded(ctxp, [&] {
        if (!ctxp || !slots || !out || n_slots < 1 || n < 0) throw ArgError("invalid reduce_slots arguments");
        if (out_mode != NBX_OUT_F32 && out_mode != NBX_OUT_F64 && out_mode != NBX_OUT_ADD_F64)
            throw ArgError("reduce_slots output mode must be F32, F64 or ADD_F64");
        Ctx* ctx = static_cast<Ctx*>(ctxp);
        NBX_CUDA(cudaSetDevice(ctx->device));
        cudaStream_t s = ctx->stream;
        const size_t bytes = (size_t)n * out_elem_bytes(out_mode);
        void* dout = out;
        if (!out_on_device) {
            ctx->out_scratch.ensure(bytes);
            dout = ctx->out_scratch.p;
            if (out_mode == NBX_OUT_ADD_F64) NBX_CUDA(cudaMemcpyAsync(dout, out, bytes, cudaMemcpyHostToDevice, s));
        }
        ctx->fault.ensure(8);
        NBX_CUDA(cudaMemsetAsync(ctx->fault.p, 0xFF, 8, s));
        NBX_CUDA(nbx::launch_reduce_slots(slots, n_slots, n, scale, out_mode, dout,
                                          static_cast<unsigned long long*>(ctx->fault.p), s));
        unsigned long long f = ~0ull;
        NBX_CUDA(cudaMemcpyAsync(&f, ctx->fault.p, 8, cudaMemcpyDeviceToHost, s));
        if (!out_on_device) NBX_CUDA(cudaMemcpyAsync(out, dout, bytes, cudaMemcpyDeviceToHost, s));
        NBX_CUDA(cudaStreamSynchronize(s));
        bad = f == ~0ull ? -1 : (int64_t)f;
        return NBX_OK;
    });
    if (st != NBX_OK) return st;
    return fault_status(ctxp, bad, first_bad);
}

// ---------------------------------------------------------------------------
// Channel-sharded image over a caller's NCCL communicator (nbx_spots_reduce).  NCCL is
// resolved at run time from the library already loaded in the process (the one that made
// the communicator: torch's bundled copy, or the caller's), so libnbx has no link-time NCCL
// dependency; ncclComm_t is an opaque pointer at this boundary.
// ---------------------------------------------------------------------------
struct NcclApi {
    int (*comm_count)(void*, int*) = nullptr;
    int (*comm_user_rank)(void*, int*) = nullptr;
    int (*reduce)(const void*, void*, size_t, int, int, int, void*, cudaStream_t) = nullptr;
    const char* (*error_string)(int) = nullptr;
};

const NcclApi* nccl_api() {
    static std::once_flag once;
    static NcclApi api;
    std::call_once(once, [] {
        void* h = nullptr;
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            h = dlopen(name, RTLD_NOW | RTLD_NOLOAD);  // the instance that created the communicator
            if (h) break;
        }
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        api.comm_count = reinterpret_cast<int (*)(void*, int*)>(dlsym(h, "ncclCommCount"));
        api.comm_user_rank = reinterpret_cast<int (*)(void*, int*)>(dlsym(h, "ncclCommUserRank"));
        api.reduce = reinterpret_cast<int (*)(const void*, void*, size_t, int, int, int, void*, cudaStream_t)>(
            dlsym(h, "ncclReduce"));
        api.error_string = reinterpret_cast<const char* (*)(int)>(dlsym(h, "ncclGetErrorString"));
    });
    return api.comm_count && api.comm_user_rank && api.reduce ? &api : nullptr;
}

constexpr int kNcclFloat64 = 8, kNcclSum = 0;  // ncclFloat64 / ncclSum (nccl.h)

int nbx_spots_reduce(void* ctxp, const nbx_spots_desc* d, int compute, void* nccl_comm, int root, int out_mode,
                     void* out, int out_on_device, int64_t* first_bad) {
    if (first_bad) *first_bad = -1;
    int rank = 0, world = 1;
    int64_t npix = 0;
    double scale = 0.0;
    int st = guarded(ctxp, [&]() -> int {
        if (!ctxp || !d) throw ArgError("NULL context or descriptor");
        if (!nccl_comm) throw ArgError("NULL NCCL communicator");
        const NcclApi* nc = nccl_api();
        if (!nc) throw ArgError("NCCL is not loaded in this process (libnccl.so.2 not found)");
        if (nc->comm_count(nccl_comm, &world) != 0 || nc->comm_user_rank(nccl_comm, &rank) != 0)
            throw ArgError("invalid NCCL communicator");
        if (root < 0 || root >= world) throw ArgError("root is not a rank of the communicator");
        if (rank == root) {
            if (out_mode != NBX_OUT_F32 && out_mode != NBX_OUT_F64 && out_mode != NBX_OUT_ADD_F64)
                throw ArgError("reduce output mode must be F32, F64 or ADD_F64");
            if (!out) throw ArgError("output buffer is NULL");
        }
        validate(d);
        const int sb = d->src_begin, se = d->src_end <= 0 ? d->n_sources : d->src_end;
        if (se - sb < world) throw ArgError("fewer sources than ranks");
        Ctx* ctx = static_cast<Ctx*>(ctxp);
        NBX_CUDA(cudaSetDevice(ctx->device));
        npix = count_pixels(d);
        // this rank's channel shard: contiguous, sizes within one, the first (n % world) one larger
        // (plan_batches, scheduler.py:138-153); the GLOBAL normalisation (kernels.py:243-245)
        nbx_spots_desc sh = *d;
        const int n = se - sb, base = n / world, extra = n % world;
        sh.src_begin = sb + rank * base + std::min(rank, extra);
        sh.src_end = sh.src_begin + base + (rank < extra ? 1 : 0);
        if (!(sh.norm > 0)) {
            double wsum = 0.0;
            for (int i = 0; i < d->n_sources; ++i) wsum += d->weights[i];
            sh.norm = wsum * (double)d->n_domains * (double)(d->oversample * d->oversample);
        }
        scale = d->r_e_sqr * d->fluence / sh.norm;
        ctx->raw_scratch.ensure((size_t)npix * sizeof(double));
        double* raw = static_cast<double*>(ctx->raw_scratch.p);
        const int s1 = nbx_spots(ctxp, &sh, compute, NBX_OUT_RAW_STORE_F64, raw, 1, nullptr);
        if (s1 != NBX_OK) return s1;
        const int r = nc->reduce(raw, raw, (size_t)npix, kNcclFloat64, kNcclSum, root, nccl_comm, ctx->stream);
        if (r != 0)
            throw CudaError(std::string("ncclReduce failed: ") + (nc->error_string ? nc->error_string(r) : "?"));
        NBX_CUDA(cudaStreamSynchronize(ctx->stream));
        return NBX_OK;
    });
    if (st != NBX_OK || rank != root) return st;
    return nbx_finalize(ctxp, static_cast<const double*>(static_cast<Ctx*>(ctxp)->raw_scratch.p), npix, scale,
                        out_mode, out, out_on_device, first_bad);
}

int nbx_add_array(void* ctxp, double* lhs, const float* rhs, int64_t n, int on_device) {
    return guarded(ctxp, [&] {
        if (!ctxp) throw ArgError("NULL context");
        if (n < 0 || (n > 0 && (!lhs || !rhs))) throw ArgError("invalid add_array arguments");
        if (n == 0) return NBX_OK;
        Ctx* ctx = static_cast<Ctx*>(ctxp);
        NBX_CUDA(cudaSetDevice(ctx->device));
        cudaStream_t s = ctx->stream;
        if (on_device) {
            NBX_CUDA(nbx::launch_add_array(lhs, rhs, n, s));
            NBX_CUDA(cudaStreamSynchronize(s));
            return NBX_OK;
        }
        DevBuf& dl = ctx->out_scratch;  // persistent scratch: a per-call cudaMalloc/cudaFree pair
        DevBuf& dr = ctx->stage_in;     // costs more than the whole kernel
        dl.ensure((size_t)n * 8);
        dr.ensure((size_t)n * 4);
        NBX_CUDA(cudaMemcpyAsync(dl.p, lhs, (size_t)n * 8, cudaMemcpyHostToDevice, s));
        NBX_CUDA(cudaMemcpyAsync(dr.p, rhs, (size_t)n * 4, cudaMemcpyHostToDevice, s));
        NBX_CUDA(nbx::launch_add_array(static_cast<double*>(dl.p), static_cast<const float*>(dr.p), n, s));
        NBX_CUDA(cudaMemcpyAsync(lhs, dl.p, (size_t)n * 8, cudaMemcpyDeviceToHost, s));
        NBX_CUDA(cudaStreamSynchronize(s));
        return NBX_OK;
    });
}

int nbx_add_noise(void* ctxp, const void* mean, void* out, int64_t n, int dtype, uint64_t seed, uint64_t image,
                  int on_device) {
    return guarded(ctxp, [&] {
        if (!ctxp) throw ArgError("NULL context");
        if (dtype != 0 && dtype != 1) throw ArgError("dtype must be 0 (f32) or 1 (f64)");
        if (n < 0 || (n > 0 && (!mean || !out))) throw ArgError("invalid noise arguments");
        if (n == 0) return NBX_OK;
        Ctx* ctx = static_cast<Ctx*>(ctxp);
        NBX_CUDA(cudaSetDevice(ctx->device));
        cudaStream_t s = ctx->stream;
        const size_t bytes = (size_t)n * (dtype ? 8 : 4);
        if (on_device) {
            NBX_CUDA(nbx::launch_noise(mean, out, n, dtype, seed, image, s));
            NBX_CUDA(cudaStreamSynchronize(s));
            return NBX_OK;
        }
        DevBuf& dm = ctx->stage_in;  // persistent scratch (see nbx_add_array)
        DevBuf& dout = ctx->out_scratch;
        dm.ensure(bytes);
        dout.ensure(bytes);
        NBX_CUDA(cudaMemcpyAsync(dm.p, mean, bytes, cudaMemcpyHostToDevice, s));
        NBX_CUDA(nbx::launch_noise(dm.p, dout.p, n, dtype, seed, image, s));
        NBX_CUDA(cudaMemcpyAsync(out, dout.p, bytes, cudaMemcpyDeviceToHost, s));
        NBX_CUDA(cudaStreamSynchronize(s));
        return NBX_OK;
    });
}

int nbx_poisson_host(const void* mean, void* out, int64_t n, int dtype, uint64_t seed, uint64_t image) {
    if (dtype != 0 && dtype != 1) return NBX_ERR_ARG;
    if (n < 0 || (n > 0 && (!mean || !out))) return NBX_ERR_ARG;
    for (int64_t p = 0; p < n; ++p) {
        const double mu = dtype ? static_cast<const double*>(mean)[p] : (double)static_cast<const float*>(mean)[p];
        const double k = nbx::poisson_draw(mu, seed, image, (uint64_t)p);
        if (dtype)
            static_cast<double*>(out)[p] = k;
        else
            static_cast<float*>(out)[p] = (float)k;
    }
    return NBX_OK;
}

int nbx_probe_fma_peak(void* ctxp, int fp64, double* tflops) {
    return guarded(ctxp, [&] {
        if (!ctxp || !tflops) throw ArgError("invalid probe arguments");
        Ctx* ctx = static_cast<Ctx*>(ctxp);
        NBX_CUDA(cudaSetDevice(ctx->device));
        int sms = 0;
        NBX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
        const int blocks = sms * 4;  // 4 x 512 threads = 2048 per SM
        DevBuf sink;
        sink.ensure(16);
        cudaStream_t s = ctx->stream;
        const int iters = fp64 ? 600 : 1200;
        NBX_CUDA(nbx::launch_fma_probe(fp64, sink.p, iters / 10, blocks, s));  // warm-up
        float best = 1e30f;
        for (int rep = 0; rep < 3; ++rep) {
            NBX_CUDA(cudaEventRecord(ctx->ev0, s));
            NBX_CUDA(nbx::launch_fma_probe(fp64, sink.p, iters, blocks, s));
            NBX_CUDA(cudaEventRecord(ctx->ev1, s));
            NBX_CUDA(cudaEventSynchronize(ctx->ev1));
            float ms = 0.f;
            NBX_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
            best = std::min(best, ms);
        }
        const double flops = 2.0 * 8 * 16 * (double)iters * blocks * 512;
        *tflops = flops / (best * 1e-3) / 1e12;
        return NBX_OK;
    });
}

}  // extern "C"
