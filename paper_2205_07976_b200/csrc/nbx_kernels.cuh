// nbx_kernels.cuh -- device-side parameter blocks shared by the kernels and
// the host runtime (nbx_runtime.cu).  Plain PODs, passed by value.
#pragma once

#include <cstdint>

namespace nbx {

// One panel as the kernel sees it: the reference's DetectorPanel
// (model.py:328-371) with the per-panel constants hoisted.
struct DevPanel {
    int32_t slow, fast;            // pixels
    int32_t thick_steps;           // >= 1
    int32_t pad0;
    int64_t out_offset;            // first output element of this panel
    double pixel_size;
    double distance;
    double bc_slow, bc_fast;       // beam_center (slow, fast)
    double fast_axis[3];
    double slow_axis[3];
    double normal[3];              // fast x slow (model.py:370-371): used for Omega
    double odet[3];                // unit normal pointing away from the sample (thickness layers)
    double thick_step;             // thickness / thick_steps (0: thin sensor)
    double inv_atten;              // 1 / attenuation_length (0 when thin)
};

// FP32 path: channels [begin, end) share the FP64 phase anchor iv0 = 1/lambda0;
// the host sorts channels by 1/lambda and cuts chunks so that
// |h_w - h_0| <= 1.5 for every reachable pixel and domain (|x| stays < 2).
struct ChunkF32 {
    double iv0;
    int32_t begin, end;
};

// FP64 path, channel-recurrence variant: sorted channels [begin, end) whose
// 1/lambda are an arithmetic progression iv0 + k*delta (to 1e-14 in phase).
// One source of the background stage: lambda, its correctly rounded reciprocal (for the
// exact division, nbx_kernels.cu:div_exact) and the weight.
struct BgChan {
    double lambda, inv_lambda, weight, pad;
};

struct RunF64 {
    double iv0, delta;
    int32_t begin, end;
};

// Everything the spot kernel reads.  All pointers are device pointers.
struct SpotsParams {
    const DevPanel* panels;
    int32_t n_panels;
    int32_t oversample;
    const double* bases;           // n_dom x 9, rows a, b, c
    int32_t n_dom;
    int32_t n_src;                 // channels in this launch (already sharded)
    const void* chan;              // FP64: double2 {1/lambda, w}; FP32: float2 {1/lambda - 1/lambda0, w}
    const ChunkF32* chunks;        // FP32 only: channel chunks sharing one phase anchor 1/lambda0
    int32_t n_chunks;
    int32_t pad1;
    const void* table;             // dense F^2 grid (FP32: scaled by sigma)
    double beam[3];
    int32_t pol_on;
    int32_t out_mode;              // NBX_OUT_*
    double n_cells_d[3];
    float n_cells_f[3];
    float n_pi_f[3];               // FP32 MUFU numerator: pi * N (rounded once, on the host)
    float pad3;
    float nnn_f;                   // Na*Nb*Nc
    double nnn_d;
    // dense-grid index: idx = (n_h - lo_h) * sH + (n_k - lo_k) * sK + (n_l - lo_l)
    int32_t lo[3];
    int32_t sH, sK;
    int32_t sh_h, sh_k;            // FP32: log2 of the power-of-two strides
    uint32_t lea_bias;             // FP32: 0x4B400000 (sH + sK + 1) mod 2^32
    double out_scale;              // r_e^2 fluence / norm (/ sigma on the FP32 path)
    double raw_scale;              // 1 / sigma (exact power of two): RAW partials are sigma-free
    void* out;
    unsigned long long* fault;     // lowest non-finite pixel (atomicMin), ~0ull when none
    int32_t max_slow, max_fast;    // launch covers rows [row0, max_slow) of every panel
    int32_t row0, pad2;            // first row of this launch (row bands of a pipelined run)
    // diffuse background (kernels.py:279-312)
    const BgChan* bg_chan;         // {lambda, 1/lambda, w} of every source
    const double* bg_stol;
    const double2* bg_fs;          // {f_bg, slope to the next point} per profile point
    int32_t n_bg_chan;
    int32_t bg_points;             // 0: no background
    double bg_scale;               // r_e^2 fluence thickness_factor / sum(w)
    unsigned long long* fault_bg;  // background stage's lowest non-finite pixel
    const RunF64* runs;            // FP64 recurrence variant: uniform channel runs (sorted channels)
    int32_t n_runs;
    int32_t pad4;
    // Sparse Fhkl (index kind 2, when the reachable Miller box is too large for a dense
    // grid): open-addressing table of packed (h, k, l) -> F^2 (x sigma on FP32), empty
    // slots ~0; misses and |index| >= 2^20 give default_f^2 (model.py:264-279).
    const unsigned long long* hash_keys;
    const void* hash_vals;         // float (FP32 path) / double (FP64 path)
    uint32_t hash_mask;            // slots - 1 (power of two)
    int32_t pad5;
    double hash_def_d;
    float hash_def_f;
    float pad6;
    unsigned long long table_tex;  // FP32 power-of-two table as a texture object (the packed loop's gather)
    const float* chunk_step;       // FP32 segmented loop: each chunk's 1/lambda step (uniform spectra)
};

}  // namespace nbx
