// Internal definitions shared by the CUDA translation units and the C-ABI layer.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "tsb.h"

namespace tsb {

constexpr int kTile = 16;          // raster CTA block edge (pixels)
constexpr int kRasterThreads = kTile * kTile;
constexpr int kMaxKeyframes = 16;
constexpr int kColorArrays = 12;  // colour SH: 48 coefficients ([c][k], splat.hpp color_sh) in 12 float4 arrays
constexpr int kMaxArrays = 3 + kMaxKeyframes + 4 + kColorArrays;  // pos_op, scale_amp, quat, motion[k], sh[4], color[12]

// Camera constants the kernels use (camera.hpp:9-49 + splat.cpp:109-111).
struct CamK {
    double fx, fy, cx, cy;
    int W, H;
    double near_plane;
    double R[9], t[3];
    double lim_x, lim_y;
    double center[3];
    // fp32 copies for the lean visibility bound (host-rounded once, not per Gaussian)
    float Rf[9], fxf, fyf, cxf, cyf, limxf, limyf, Wf, Hf;
};

// Render options (splat.hpp:28-37) in the forms the kernels compare against.
constexpr float kCoarseMaha = 1e-3f;       // relative window that triggers the precise bound
constexpr float kCoarseAlpha = 1e-4f;
struct OptK {
    double alpha_thr, floor_T, dilation, sigma_cutoff, cov_eps, cut2;
    int ts;            // binning tile size
    int tiles_x, tiles_y;
    int sub;           // 16x16 raster blocks per tile edge = ceil(ts/16)
    float alpha_thr_f, floor_f, cut2_f, cov_eps_f;
    float dilation_f, sigma_cutoff_f;
    int dist;          // distortion channel: accumulate the shifted depth moments
    int exact;         // TSB_CH_EXACT: every pixel goes to the fp64 fix-up
    float trel_flag;   // relative T error bound above which a pixel is recomposited (fix-up reason 8)
    // the raster's decision thresholds (host-computed: constant-bank operands in the hot loop,
    // no registers): coarse windows, the clearly-outside maha, the prefilter edges
    float coarse_m_f, coarse_a_f, outside_f, m_lo_f, a_hi_f;
    double bg_quad[8];
    double bg_phasor[4];
    double bg_color[3];
};

// Device-resident scene (fp32 SoA float4 arrays; see tsb.h for the mapping).
struct SceneK {
    int n, nk, nf, sh_degree;
    double freq[2], s_int, c;
    const float4* pos_op;     // x, y, z, opacity_logit
    const float4* scale_amp;  // log_scale xyz, reflectivity_dc
    const float4* quat;       // w, x, y, z
    const float4* motion;     // [nk][n] keyframe offsets (xyz, 0)
    const float4* sh;         // [4][n] reflectivity SH coefficients 1..15 (+pad); null when sh_degree == 0
    const float4* color_sh;   // [12][n] colour SH, flat coefficient 16 c + k in array (16 c + k) / 4; null: no colour
    // Time-independent per-Gaussian cache, refreshed whenever the parameters change
    // (tsb_scene_set_params, Adam): cov3d = M3 M3^T (6 planes xx, xy, xz, yy, yz, zz)
    // and opacity = sigmoid(logit), computed by the same fp64 code prep64 used inline,
    // so every frame of a sweep reads them instead of recomputing.  Null: inline.
    const double* cov6;
    const double* opac;
    const float* cov6f;  // fp32 copy of cov6 (lean visibility bound) or null
};

struct FrameK {
    int key;
    double w;
};

// Per-frame values the forward kernels read from device memory (so one captured
// CUDA graph serves every frame): written by a host->device copy from the pass's
// pinned staging slot at the start of each forward.
struct FrameDev {
    FrameK F;
    const float* target;  // loss target (planar [4*nf][H][W]) or null
    int stamp;            // fix-up record-cache stamp
    int pad;
};

// fp32 raster records, indexed by Gaussian (SoA).  The conic is stored
// factored, conic = L^T L, L = [[l11, l12], [0, l22]] (see tsb_raster.cu).
struct RecK {
    float4* A;  // base_x, base_y (integer rect origin), mean.x - base_x, mean.y - base_y
    float4* B;  // l11, l12, l22, opacity
    float4* C;  // coef, depth, sin(psi_0), cos(psi_0)
    float4* D;  // sin(psi_1), cos(psi_1), 0, 0   (second frequency only)
    const uint2* rect;  // alias of the pass's tile rects: (x0 | x1 << 16, y0 | y1 << 16)
};

// Equal-key runs of the depth sort, resolved by the readers of the order (tsb_ties.cuh).
struct TieK {
    const uint32_t* keys;    // sorted compressed depth keys; null: the order is already exact
    const double* depth64;   // fp64 depth per Gaussian
    int32_t* abort;          // frame abort word (bit 1: a run longer than kMaxTieRun)
};

// The frame's depth order as the raster kernels read it.  There are no per-tile
// lists: the rank-order arrays are scanned by every raster block, which keeps the
// ranks whose tile rect covers its tile -- exactly the reference's tile list
// (splat.cpp:187-200, bbox tile ranges in global (depth, index) order) -- up to the
// point where all its pixels have terminated (SURVEY finding 1: ~1 % of a list).
//   ord[r]   Gaussian at rank r < *n_rank of the exact order (tsb_ties.cuh resolved)
//   trect[r] its tile rect, (tx0 | tx1 << 16, ty0 | ty1 << 16)
constexpr int kBlkListCap = 4096;  // list entries a raster block records for its backward
struct ScanK {
    const uint32_t* ord;
    const uint2* trect;
    const int32_t* n_rank;   // ranks in the order (the prefix end under the prefix sort)
    const int32_t* n_all;    // visible Gaussians
    int2* blk_term;          // per raster block: (rank after its last scanned pass, entries before that rank)
    uint32_t* blk_list;      // per raster block: the ranks of the first kBlkListCap entries of its list, as
                             // the forward consumed them (the backward walks them back instead of rescanning)
    int32_t* abort;          // frame abort word (bit 3: the prefix ended with a pixel alive)
    unsigned long long* work;  // profiling: [0] evaluations, [1] contributions (null: not counted)
    // Deterministic backward (TSB_CH_DETERMINISTIC): a private partial-sum slot per (rank, tile
    // of its rect, raster sub-block), reduced per Gaussian in a fixed order; null: atomics.
    const uint32_t* det_off;   // [n_rank + 1] first slot of each rank (rect area x sub-blocks, scanned)
    float* det_part;           // [slots][8]
    int nsub2;                 // raster blocks per tile
    // Super-tile lists: the ranks whose tile rect meets each super-tile (2^sup_log x 2^sup_log
    // tiles), in rank order, with their rects.  A block scans its super-tile's list instead of
    // the whole order; scan positions (blk_term.x, FixState::r_end) index that list.  Null
    // sl_off (a short order, kSlMinRanks): blocks scan the order itself (positions = ranks).
    const uint32_t* sl_off;    // [nsup + 1]
    const uint32_t* sl_rank;   // [sl_cap] (null without lists)
    const uint2* sl_rect;      // [sl_cap] (trect without lists)
    int sup_x, sup_log;
};
// One tile's scan list: its offset in the super-tile lists and its length (two 32-bit
// values: the list pointers stay kernel parameters, not live registers of the scan loops).
struct ScanSeg {
    uint32_t off;
    int n;
};
__device__ __forceinline__ ScanSeg scan_seg(const ScanK& sc, int tx, int ty) {
    if (!sc.sl_off) return ScanSeg{0u, *sc.n_rank};  // short order: the order itself
    const int s = (ty >> sc.sup_log) * sc.sup_x + (tx >> sc.sup_log);
    const uint32_t a = sc.sl_off[s], b = sc.sl_off[s + 1];
    return ScanSeg{a, (int)(b - a)};
}
// The tile rect / rank at scan position p (without lists sl_rect is trect and sl_rank null).
__device__ __forceinline__ uint2 seg_rect(const ScanK& sc, const ScanSeg& sg, int p) { return sc.sl_rect[sg.off + p]; }
__device__ __forceinline__ uint32_t seg_rank(const ScanK& sc, const ScanSeg& sg, int p) {
    return sc.sl_rank ? sc.sl_rank[sg.off + p] : (uint32_t)p;
}
// Build arguments of the super-tile lists (k_order_ranks counts + scan, k_sl_emit).
constexpr int kSlChunk = 256;     // ranks per chunk
constexpr int kSlMinRanks = 32768; // orders up to this long are scanned directly (no lists)
constexpr int kSlMaxSup = 1024;   // super-tiles per frame (the super-tile grows past this)
constexpr int kSlMaxSupSide = 64; // super-tiles per row / column (likewise)
constexpr int kSlMaxBlocks = 148 * 8;  // blocks building the lists (contiguous rank ranges each)
struct SuperK {
    uint32_t* hist;      // [nsup][hist_stride] per-block pair counts -> offsets within the row
    int hist_stride;     // histogram columns = the build grid's upper bound (kSlMaxBlocks)
    uint32_t* row_total; // [nsup] pairs per super-tile
    uint32_t* off;       // ScanK::sl_off
    uint32_t* rank;      // ScanK::sl_rank
    uint2* rect;         // ScanK::sl_rect
    int cap;             // entries the lists can hold; more: abort bit 1, the total in *total
    int32_t* total;
    int sup_x, sup_log, nsup;
    unsigned long long* work;  // profiling: [2] += ranks, [3] += list entries (null: not counted)
};
// The slot of (rank r with tile rect tr, tile (tx, ty), raster sub-block sb).
__device__ __forceinline__ size_t det_slot(const ScanK& sc, int r, uint2 tr, int tx, int ty, int sb) {
    const int tx0 = tr.x & 0xffff, w = (int)(tr.x >> 16) - tx0 + 1, ty0 = tr.y & 0xffff;
    return (size_t)sc.det_off[r] + ((size_t)(ty - ty0) * w + (tx - tx0)) * sc.nsub2 + sb;
}
// Block-uniform test of a frame abort word.  Kernels raise the word while other blocks of
// the same launch are starting (the raster's bit 8, the tie reader's bit 2, ...), so the
// threads of one block could read different values; the exit decision -- and with it every
// barrier and warp collective that follows -- must be the block's.
__device__ __forceinline__ bool block_aborted(const int32_t* a) {
    return __syncthreads_or(a != nullptr && *reinterpret_cast<const volatile int32_t*>(a) != 0);
}
__device__ __forceinline__ bool tile_covers(uint2 tr, int tx, int ty) {
    return (int)(tr.x & 0xffffu) <= tx && tx <= (int)(tr.x >> 16) && (int)(tr.y & 0xffffu) <= ty &&
           ty <= (int)(tr.y >> 16);
}

// Per-pixel raster state written by the forward pass for the backward pass.
struct PixK {
    float* out;          // [C][H][W] planar outputs: quad(4*nf), depth_raw, depth, weight, T, phasor(2*nf), distortion
    double* dist3;       // [3][H][W] distortion moments about the pixel's first contributor depth (fp64):
                         //   dref, SDs = sum w (d - dref), SD2s = sum w (d - dref)^2 (null: not computed)
    int32_t* n_contrib;  // may be null
    int32_t* n_processed;
    int32_t* last;       // entries of the tile list the backward walks (bit 31: fp64-fixed)
    float* T_pre;        // T before the last contributor
    float* d_quad;       // [4*nf][H][W] upstream (written by loss epilogue)
    int32_t* flagged;    // list of fp64-fixup pixels
    double* out64;       // TSB_CH_EXACT: fp64 copy of `out` (written by k_fixup) or null
    int32_t* n_flagged;  // device counter
    const int32_t* abort;  // frame abort word (overflow / long tie run): later kernels do nothing
};

// Per-channel loss weights, passed by value (no staging copy, no host sync).
struct ChW {
    float w[8];
};

inline int out_channels(int nf) { return 6 * nf + 5; }
// Channel plane index inside PixK::out.
__host__ __device__ inline int ch_depth_raw(int nf) { return 4 * nf; }
__host__ __device__ inline int ch_depth(int nf) { return 4 * nf + 1; }
__host__ __device__ inline int ch_weight(int nf) { return 4 * nf + 2; }
__host__ __device__ inline int ch_T(int nf) { return 4 * nf + 3; }
__host__ __device__ inline int ch_phasor(int nf) { return 4 * nf + 4; }
__host__ __device__ inline int ch_distortion(int nf) { return 6 * nf + 4; }

// Upstream images of BufferGrads (splat.hpp:73-77); null = channel skipped.
struct UpK {
    const float* quad;        // [4*nf][H][W]
    const float* phasor;      // [2*nf][H][W]
    const float* depth_raw;   // [H][W]
    const float* weight;
    const float* distortion;
    const float* transm;
    const float* color;       // [3][H][W] colour (TSB_CH_COLOR)
    const float* mf;          // [3][H][W] motion_fwd_acc (TSB_CH_FLOW)
    const float* mb;          // [3][H][W] motion_bwd_acc
};
// Scene statistics buffer: background gradients (quad 4*nf, then phasor 2*nf) and the loss.
constexpr int kStatBg = 0, kStatLoss = 12, kStatBgColor = 13, kStats = 16;

// ---- launchers (defined in the .cu files) ----
// tsb_geom.cu (fp64, compiled without FMA contraction)
void launch_preprocess(const SceneK& S, const CamK& C, const OptK& O, const FrameDev* F,
                       uint32_t* depth_key, double* depth64, uint32_t* gidx, uint32_t* touched, uint2* rect,
                       RecK rec, int32_t* n_visible, uint32_t* key_range, bool lean, cudaStream_t st);
// depth64 / rect / raster records of list[0, *count) (a lean frame's sorted prefix), or of
// every visible Gaussian plus the identity order when list is null.  Returns launches.
int launch_records(const SceneK& S, const CamK& C, const OptK& O, const FrameDev* F, const uint32_t* list,
                   const int32_t* count, int n, const uint32_t* depth_key, double* depth64, uint32_t* gidx,
                   uint2* rect, RecK rec, int32_t* abort, cudaStream_t st);
// fp64 record cache for the fix-up (valid when stamp[g] == frame stamp).
struct Rec64 {
    double4 m0;  // mean x, mean y, conic a, conic b
    double4 m1;  // conic c, opacity, coef, depth
    int4 rect;   // x0, x1, y0, y1
};

// fp64 end state of a recomposited pixel (k_fixup), what its fp64 backward (k_fixup_bwd)
// needs: T_N, T before the last contributor (before the alpha == 1 entry when T hit 0),
// sum w, the distortion moments about the first contributor's depth, and where its walk
// stopped: the rank after its last processed entry and the entries processed.
struct FixState {
    double T, Tpre, SW, dref, SDs, SD2s;
    int r_end, e_end;
};
// The bound of T's relative error (first order, worst case: linear in the number of
// contributions) above which a pixel is recomposited in fp64: an almost opaque splat
// (1 - alpha lost to fp32 rounding) makes T -- and every later weight -- inaccurate.
constexpr float kTrelFlag = 1e-4f;
constexpr int kFixStateCap = 1 << 16;  // recomposited pixels per frame with an fp64 backward
constexpr int kLastFixed = (int)0x80000000;  // PixK::last bit 31: pixel recomposited in fp64
constexpr int kLastBwd64 = 0x40000000;       // bit 30: its backward runs in fp64 (k_fixup_bwd)
constexpr int kLastMask = 0x3fffffff;

struct FixupK {
    ScanK sc;          // the order the walk scans (ranks whose rect covers the pixel's tile)
    int32_t* overflow;
    int* stamp;        // [n] frame stamp of the cached record (FrameDev::stamp)
    int* work;         // [n] Gaussians queued for the record cache
    int* work_n;
    Rec64* cache;      // [n]
    FixState* state;   // [state_cap] per flagged pixel (fix-up slot): fp64 state for k_fixup_bwd
    int state_cap;
    int* fix_idx;      // [npx] fix-up slot of a recomposited pixel (the deterministic backward's lookup)
};
int launch_fixup(const SceneK& S, const CamK& C, const OptK& O, const FrameDev* fd, const FixupK& fx,
                 const PixK& px, int nf, cudaStream_t st);  // returns kernels launched
void launch_fixup_bwd(const SceneK& S, const CamK& C, const OptK& O, const FrameDev* fd, const FixupK& fx,
                      const PixK& px, const UpK& up, int nf, double* screen, int scap, cudaStream_t st);
// deterministic: the same per pixel, one warp per raster block in pixel order, into the slots
void launch_fixup_bwd_det(const SceneK& S, const CamK& C, const OptK& O, const FrameDev* fd, const FixupK& fx,
                          const PixK& px, const UpK& up, int nf, cudaStream_t st);
void launch_chain(const SceneK& S, const CamK& C, const OptK& O, const FrameK& F,
                  const uint32_t* touched, double* screen, float4* grads, cudaStream_t st);
void launch_param_cache(const SceneK& S, double* cov6, double* opac, float* cov6f, cudaStream_t st);
constexpr size_t kPcacheWords = 10;  // doubles per Gaussian of the parameter cache (7 fp64 + 6 fp32 words)
// tsb_bin.cu
// tsb_sort.cu: hand-written onesweep LSD radix sort of 32-bit keys + values (4 passes);
// the result is back in (keys_a, vals_a).  Returns the number of kernels launched.
size_t radix_sort_scratch_words(int n);
int radix_sort32(uint32_t* keys_a, uint32_t* keys_b, uint32_t* vals_a, uint32_t* vals_b, int n, uint32_t* scratch,
                 cudaStream_t st);
// 3 passes over keys compressed to 24 bits with the device-side key range
// (range[0] = min, range[1] = max); result in (keys_b, vals_b).
int radix_sort24(uint32_t* keys_a, uint32_t* keys_b, uint32_t* vals_a, uint32_t* vals_b, int n, uint32_t* scratch,
                 const uint32_t* range, cudaStream_t st);
// Nearest-prefix order (tsb_sort.cu): sorts only ranks [0, *n_bin) of the order,
// n_bin <= cap, into (keys_out, vals_out); keys stay intact; raises abort bit 3 when
// even the nearest top digit exceeds cap.
size_t prefix_sort_scratch_words(int cap);
int radix_sort24_prefix(const uint32_t* keys, uint32_t* keys_out, uint32_t* vals_out, uint32_t* tmp_keys,
                        uint32_t* tmp_vals, int n, int cap, uint32_t* scratch, uint32_t* ps, const uint32_t* range,
                        const int32_t* n_visible, int32_t* n_bin, int32_t* abort_word, cudaStream_t st);
// Global (depth, index) order: stable sort on compressed fp32 depth keys; runs of equal
// keys are ordered by the fp64 depth where the order is read (sorted_at, tsb_ties.cuh).
int launch_sort_depth(uint32_t* keys_a, uint32_t* keys_b, uint32_t* vals_a, uint32_t* vals_b,
                      const uint32_t* key_range, int n, uint32_t* scratch, cudaStream_t st);  // -> (keys_b, vals_b)
// out[r] = Gaussian at rank r of the exact order, r < *n_visible (debug / parity copies)
void launch_materialize_order(const uint32_t* sorted, const TieK& T, const int32_t* n_visible, int n, uint32_t* out,
                              cudaStream_t st);
int launch_sort_depth64(const double* depth64, const uint32_t* touched, uint32_t* keys_a, uint32_t* keys_b,
                        uint32_t* vals_a, uint32_t* vals_b, int n, uint32_t* scratch, cudaStream_t st);
// ord / trect of ranks r < *n_rank (the raster kernels' scan arrays, ScanK)
// + the super-tile lists (3 kernels; returns the launch count); n: upper bound of *n_rank
int launch_order_ranks(const uint32_t* sorted, const TieK& T, const uint2* rect, int ts, const int32_t* n_rank,
                       int n, uint32_t* ord, uint2* trect, const SuperK& sk, cudaStream_t st);
// deterministic backward: slot offsets of the ranks (device scan; writes det_off[0..V]) and
// the fixed-order reduction of the slots into the screen-space gradients (+=)
void launch_det_offsets(const ScanK& sc, uint32_t* det_off, uint32_t* total, cudaStream_t st);
void launch_det_reduce(const ScanK& sc, int n, double* screen, int scap, cudaStream_t st);
// parity / debug: the reference's complete tile lists (splat.cpp:187-200) from the scan arrays
void launch_tile_counts(const ScanK& sc, int tiles_x, int ntiles, uint32_t* counts, cudaStream_t st);
void launch_tile_lists(const ScanK& sc, int tiles_x, int ntiles, const int64_t* offsets, uint32_t* ids,
                       cudaStream_t st);
// tsb_raster.cu
void raster_init();  // kernel attributes; call before any capture
void launch_raster_fwd(const RecK& rec, const ScanK& sc, const OptK& O, int W, int H, int nf, PixK px,
                       const FrameDev* fd, bool loss, const ChW& ch_w, double* loss_part, cudaStream_t st);
void launch_fixup_loss(const PixK& px, int W, int H, int nf, const FrameDev* fd, const ChW& ch_w,
                       double* loss_extra, bool deterministic, cudaStream_t st);
void launch_raster_bwd(const RecK& rec, const ScanK& sc, const OptK& O, int W, int H, int nf, const float* dpsi,
                       PixK px, const UpK& up, double* screen, int scap, double* bg_part, cudaStream_t st);
// out[c] = (out[c] + sum_i part[i][c]) * scale; nothing when *abort != 0 (abort may be null).
void launch_reduce_partials(const double* part, int nparts, int width, double* out,
                            double scale, const int32_t* abort, cudaStream_t st);
// tsb_mlp.cu: tcgen05 (kind::tf32, 3xTF32) GEMM with strided operands and fused epilogue.
struct GemmArgs {
    const float* A;  // A(m, k) = A[m * a_m + k * a_k]
    int64_t a_m, a_k;
    const float* B;  // B(n, k) = B[n * b_n + k * b_k]
    int64_t b_n, b_k;
    int M, N, K;      // N <= 128
    int k_per_slice;  // split-K slice length (multiple of 32); grid.y = slices
    float* C;         // C[slice * slice_stride + m * ldc + n]
    int64_t ldc, slice_stride;
    const float* bias;  // [N] or null
    int relu;
    const float* mask;  // C *= (mask[m * ldmask + n] > 0) when non-null
    int64_t ldmask;
    float* rowsum;      // [slice][M]: sum over this slice's k of A(m, k) (row-contiguous A only), or null
    const uint32_t* maskbits;  // instead of mask: C *= bit n of maskbits[m * ldmaskbits + n / 32], or null
    int64_t ldmaskbits;
    // DeformNet input-gradient chain fused into the epilogue (l_x = 10 encodings): instead of
    // storing C, chain_dpos[m * chain_pstride + c] (+)= sum_j gamma'_j(v_c) C[m][21 c + j] *
    // chain_inv_scale with v_c = chain_x[m * chain_ldx + 21 c] (launch_gemm_tf32x3 returns
    // kGemmNoChain when the launch cannot fuse it)
    const float* chain_x;
    int64_t chain_ldx, chain_pstride;
    double chain_inv_scale;
    float* chain_dpos;
    int chain_acc;
};
constexpr int kGemmNoChain = -2;
int launch_gemm_tf32x3(const GemmArgs& g, int slices, cudaStream_t st);  // kernels launched (0, 1; -1: N > 128)
void launch_reduce_slices(const float* part, int slices, int64_t stride, int64_t n, float* out, bool accumulate,
                          cudaStream_t st);
// DeformNet (tsb_mlp.cu): time encoding values (computed on the host in fp64), helpers.
struct DeformEnc {
    int n;
    float v[64];
};
constexpr int kMlpMaxLayers = 9;  // 8 hidden + output
struct MlpLayout {
    int layers;       // hidden + 1
    int total_chunks; // sum of chunks
    int rows[kMlpMaxLayers], cols[kMlpMaxLayers], nt[kMlpMaxLayers], chunks[kMlpMaxLayers],
        cols_pad[kMlpMaxLayers];
    int64_t w_off[kMlpMaxLayers], b_off[kMlpMaxLayers], chunk_off[kMlpMaxLayers];  // floats / floats / bytes
};
struct MlpFwdArgs {
    MlpLayout lay;
    const float* pos;
    int64_t pos_stride, n;
    double inv_scale;
    int l_x, din;
    DeformEnc te;
    const char* wpack;
    const float* params;
    float* X;  // encodings [n][ldx] (nullable)
    int64_t ldx;
    float* H[kMlpMaxLayers];  // hidden activations [n][ldh] (nullable)
    uint32_t* Hbits[kMlpMaxLayers];  // their ReLU gates, 1 bit per unit: [n][ldh / 32] words (nullable)
    int64_t ldh;
    float* out;
    int64_t out_stride;
};
void launch_pack_weights(const MlpLayout& lay, const float* params, char* out, cudaStream_t st);
void launch_mlp_fwd_fused(const MlpFwdArgs& a, cudaStream_t st);
void launch_deform_encode(const float* pos, int64_t pos_stride, int64_t n, double inv_scale, int l_x,
                          const DeformEnc& te, float* X, int64_t ldx, cudaStream_t st);
void launch_deform_chain(const float* d_input, int64_t ldd, const float* X, int64_t ldx, int64_t n, double inv_scale,
                         int l_x, float* d_pos, int64_t dpos_stride, bool accumulate, cudaStream_t st);
// tsb_ssim.cu: lambda's part of the trainer image loss for the quad channels.
struct SsimArgs {
    int nz;                  // channels with a non-zero SSIM weight
    int chans[8];            // their quad channel indices
    double scale[8];         // d_quad[c] += scale * dS/dx:  -w_c lambda / npx
    double lam_w[8];         // loss += lam_w (1 - mean S):  w_c lambda
    double* g;               // [nz][3][H][W] gradient planes
    double* part;            // [nz][blocks] partial sums of S
    float* d_quad;
    double* loss;
    const int32_t* abort;
    const FrameDev* fd;      // the frame's target (fd->target)
};
void ssim_init();  // window constants (outside any stream capture)
int ssim_blocks(int W, int H);
void launch_ssim(const float* x, int W, int H, const SsimArgs& a, cudaStream_t st);
// tsb_densify.cu: densification surgery (trainer.cpp:385-470).
struct DensifyK {
    const float* grad_sum;  // densify statistic: sum of |dL/dx_canon| per Gaussian
    int64_t count;          // iterations accumulated
    double grad_threshold, opacity_floor, split_scale /* fraction x scene extent */, split_shrink;
    int min_count;
};
struct DensifyScratch {
    uint32_t *transparent, *tprefix, *keep, *extra, *kpos, *epos, *scan_tmp, *totals;  // totals: kept, extra, transp
    uint8_t* decision;
};
void launch_densify_plan(const SceneK& S, const DensifyK& D, DensifyScratch& w, cudaStream_t st);
void launch_densify_scatter(const SceneK& S, const DensifyK& D, const DensifyScratch& w, uint32_t n_kept, int narrays,
                            const float4* P, const float4* M, const float4* V, float4* P2, float4* M2, float4* V2,
                            int n_new, cudaStream_t st);
// tsb_ext.cu: colour and flow channels (splat.cpp:273-334 forward, 361-505 backward, 560-571 chain).
constexpr int kExtPlanes = 15;  // colour 3, motion_fwd_acc 3, motion_bwd_acc 3, flow_fwd 2, flow_bwd 2, flow_valid 2
struct ExtK {
    float4* col;          // [n] clamped colour of the frame (rgb, 0); null: no colour channel
    const float4* mf;     // [n] motion_fwd (xyz, 0) or null (zero)
    const float4* mb;     // [n] motion_bwd or null
    float* out;           // [kExtPlanes][H][W]
    double* out64;        // TSB_CH_EXACT: [9][H][W] fp64 colour / motion accumulators or null
    float* screen;        // [9][n] per-Gaussian d_color, d_motion_fwd, d_motion_bwd (summed over pixels)
    float4* d_motion;     // [2][n] SceneGrads::d_motion_fwd / d_motion_bwd of the last backward
    double* bg_part;      // [blocks][3] d_bg_color partials
    int flow;             // flow outputs requested
};
void launch_ext_prep(const SceneK& S, const CamK& C, const FrameDev* fd, const uint32_t* touched, const ExtK& E,
                     const int32_t* abort, cudaStream_t st);
void launch_ext_fwd(const RecK& rec, const SceneK& S, const CamK& C, const OptK& O, const FrameDev* fd,
                    const ScanK& sc, const FixupK& fx, const PixK& px, int nf, const ExtK& E, cudaStream_t st);
void launch_ext_bwd(const RecK& rec, const OptK& O, int W, int H, int nf, const ScanK& sc, const PixK& px,
                    const UpK& up, const ExtK& E, double* screen, int scap, cudaStream_t st);
// flow_loss (losses.cpp:168-251) on the rendered flow channels; 3 kernels.
struct FlowK {
    const float* target[2];  // [3][H][W] (u, v, valid) per direction, null = absent
    float* d_macc;           // [6][H][W]: d_motion_fwd_acc, d_motion_bwd_acc (scaled by the loss weight)
    double* part;            // [flow_loss_parts][4]
    double* res;             // [4]: value, valid pixels, gradient scale fwd / bwd (0: no gradient)
    const int32_t* abort;
};
int flow_loss_parts(int npx);
// render-stack planes (eval.cpp:96-121): [0] depth gated at weight > 0.5, [1] d_ToF from the quad
void launch_stack_planes(const float* out, int nf, int npx, double freq, double c, float* dst, cudaStream_t st);
void launch_flow_loss(const CamK& C, int nf, const float* out_tof, const float* ext, const FlowK& F, double weight,
                      cudaStream_t st);
void launch_chain_ext(const SceneK& S, const CamK& C, const FrameK& F, const uint32_t* touched, const ExtK& E,
                      float4* grads, cudaStream_t st);
// tsb_optim.cu
void launch_pack_params(float4* dst, const float* src, int n, int comps, int comp0, int ncomp_dst,
                        cudaStream_t st);
void launch_unpack(const float4* src, float* dst, int n, int comps, int comp0, cudaStream_t st);
// SH coefficients 1..15 of a [n][16] host-layout array <-> the 4 float4 SH arrays
void launch_pack_sh(float4* dst4, float4* scale_amp, const float* src16, int n, cudaStream_t st);
void launch_unpack_sh(const float4* src4, float* dst16, int n, cudaStream_t st);
// [n][4 * na] host-layout rows <-> na float4 arrays (colour SH: na = 12; motions: na = 1 with 3 comps)
void launch_pack_rows(float4* dst, const float* src, int n, int na, int comps, cudaStream_t st);
void launch_unpack_rows(const float4* src, float* dst, int n, int na, int comps, cudaStream_t st);
void launch_adam(float4* params, float4* grads, float4* m, float4* v, int n, int narrays,
                 const double* lr4 /* host [narrays*4] */, double beta1, double beta2, double eps,
                 double bc1, double bc2, float* densify, cudaStream_t st);

void launch_adam_flat(float* p, const float* g, float* m, float* v, size_t n, double lr, double b1, double b2,
                      double eps, double bc1, double bc2, cudaStream_t st);
void launch_adam_reindex(const float* m, const float* v, const int32_t* src, size_t n_new, int stride, float* m2,
                         float* v2, cudaStream_t st);

}  // namespace tsb
