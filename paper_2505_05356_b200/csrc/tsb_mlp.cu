// DeformNet (deform.hpp:19-66, deform.cpp:28-159) on the 5th-generation tensor cores.
//
// The one dense contraction of the system: an MLP mapping (canonical position,
// time) -> position offset.  Every layer is a tcgen05 GEMM
//     D[128-row tile x N] = sum_k A(m, k) B(n, k)      (fp32 accumulator in TMEM)
// issued by one thread with kind::tf32 operands staged in shared memory in the
// canonical K-major no-swizzle layout (8-row x 16-byte core matrices).  The
// reference computes in fp64; to stay within the parity tolerances the operands
// are split 3xTF32 (a = a_hi + a_lo, both tf32; D += a_hi b_hi + a_hi b_lo +
// a_lo b_hi), which keeps ~fp32 accuracy at a third of the tf32 tensor rate.
// Operands are read through generic (m, k) / (n, k) strides, so the same kernel
// serves the input gradient (delta W) and the weight gradient (delta^T H, split over
// row slices) without transposes in memory: raw fp32 chunks stream into a ring of
// shared-memory stages several chunks ahead (cp.async, or one TMA bulk copy per operand
// when a chunk is a contiguous run of full-width rows), every thread splits one chunk
// into the hi / lo tiles (transposed operands are transposed on that read), and a
// constant B operand is split once per CTA and kept resident.  The epilogue (TMEM ->
// registers) fuses bias, ReLU and the ReLU-gate mask.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

#include "tsb_internal.h"

namespace tsb {

namespace {

constexpr int kGemmThreads = 512;  // 16 warps stage; thread 0 issues MMAs; warps read TMEM by lane quadrant
constexpr int kGemmM = 128;        // rows per tile (TMEM lanes)
constexpr int kGemmKc = 32;        // K elements staged per round (8 core-matrix columns of 4 tf32)
constexpr uint32_t kCoreBytes = 128;                       // 8 rows x 16 B
constexpr uint32_t kGroupBytes = (kGemmKc / 4) * kCoreBytes;  // one 8-row group across the K chunk

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// Shared-memory matrix descriptor (tcgen05), K-major, no swizzle:
// LBO = byte step between core matrices along K, SBO = between 8-row groups.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version 1 (sm_100); base offset 0, SWIZZLE_NONE
    return d;
}

// Instruction descriptor: D f32, A/B tf32, both K-major, M x N.
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t* mbar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(mbar))
                 : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* mbar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mbar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* mbar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE_%=;\n\t"
        "bra WAIT_%=;\n\t"
        "DONE_%=:\n\t}" ::"r"(smem_u32(mbar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_after_sync() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_before_sync() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

// 3xTF32 split: hi = a rounded (half away from zero) to tf32 -- its 13 low mantissa bits
// zero, by integer add + mask (finite inputs; cvt.rna.tf32 is an emulated sequence on
// sm_100), lo = a - hi (exact in fp32).  The tensor core reads the fp32 bit patterns and
// ignores the 13 low mantissa bits, so lo enters truncated to tf32: |error| <= 2^-21 |a|.
__device__ __forceinline__ void split_tf32(float a, float& hi, float& lo) {
    hi = __uint_as_float((__float_as_uint(a) + 0x1000u) & 0xffffe000u);
    lo = a - hi;
}

// Byte offset of element (row r, k) in a K-major no-swizzle tile of the K chunk.
__device__ __forceinline__ uint32_t core_off(int r, int k) {
    return (uint32_t)(r >> 3) * kGroupBytes + (uint32_t)(k >> 2) * kCoreBytes + (uint32_t)(r & 7) * 16u +
           (uint32_t)(k & 3) * 4u;
}

// Stage rows [r0, r0 + R) x k [k0, k0 + kGemmKc) of X(r, k) = P[r * sr + k * sk]
// (zero outside rows < nrows, k < kend) into hi / lo tiles.  Fast paths: 16-byte loads
// along K (one core-matrix row, stored whole; consecutive threads take consecutive rows
// of a core matrix, so the shared stores are conflict-free) or along rows (transposed
// operands: four rows of one k per load).
__device__ __forceinline__ void split4(const float4 v, float4& h, float4& l) {
    split_tf32(v.x, h.x, l.x);
    split_tf32(v.y, h.y, l.y);
    split_tf32(v.z, h.z, l.z);
    split_tf32(v.w, h.w, l.w);
}

__device__ __forceinline__ void stage_tile(const float* __restrict__ P, int64_t sr, int64_t sk, int r0, int nrows,
                                           int k0, int kend, int R, char* hi, char* lo) {
    const bool aligned = ((uintptr_t)P & 15) == 0;
    if (sk == 1 && (sr & 3) == 0 && aligned && k0 + kGemmKc <= kend) {
        for (int idx = threadIdx.x; idx < R * (kGemmKc / 4); idx += kGemmThreads) {
            const int r8 = idx & 7, q = (idx >> 3) & 7, rg = idx >> 6;
            const int r = rg * 8 + r8, gr = r0 + r;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (gr < nrows) v = __ldg(reinterpret_cast<const float4*>(P + (int64_t)gr * sr + k0 + 4 * q));
            float4 h, l;
            split4(v, h, l);
            const uint32_t o = core_off(r, 4 * q);
            *reinterpret_cast<float4*>(hi + o) = h;
            *reinterpret_cast<float4*>(lo + o) = l;
        }
        return;
    }
    if (sr == 1 && (sk & 3) == 0 && aligned && r0 + R <= nrows && (r0 & 3) == 0) {
        const int rq_n = R / 4;
        for (int idx = threadIdx.x; idx < kGemmKc * rq_n; idx += kGemmThreads) {
            const int k = idx / rq_n, rq = idx - k * rq_n, gk = k0 + k;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (gk < kend) v = __ldg(reinterpret_cast<const float4*>(P + (r0 + 4 * rq) + (int64_t)gk * sk));
            float4 h, l;
            split4(v, h, l);
            const float hv[4] = {h.x, h.y, h.z, h.w}, lv[4] = {l.x, l.y, l.z, l.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint32_t o = core_off(4 * rq + i, k);
                *reinterpret_cast<float*>(hi + o) = hv[i];
                *reinterpret_cast<float*>(lo + o) = lv[i];
            }
        }
        return;
    }
    const bool kcontig = sk == 1;
    for (int idx = threadIdx.x; idx < R * kGemmKc; idx += kGemmThreads) {
        int r, k;
        if (kcontig) {
            r = idx / kGemmKc;
            k = idx - r * kGemmKc;
        } else {
            k = idx / R;
            r = idx - k * R;
        }
        const int gr = r0 + r, gk = k0 + k;
        const float v = (gr < nrows && gk < kend) ? P[(int64_t)gr * sr + (int64_t)gk * sk] : 0.f;
        float h, l;
        split_tf32(v, h, l);
        const uint32_t o = core_off(r, k);
        *reinterpret_cast<float*>(hi + o) = h;
        *reinterpret_cast<float*>(lo + o) = l;
    }
}

}  // namespace

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Accumulation precision: the tensor core's fp32 accumulation error grows linearly
// with the number of K steps (measured: 2e-6 of the result's scale per 256 rows of a
// delta^T H reduction, 5e-4 per 65,536).  FLUSH kernels (the weight-gradient
// reductions over all rows) therefore restart the TMEM accumulator every
// kFlushChunks K chunks and add it into round-to-nearest fp32 registers.
constexpr int kFlushChunks = 8;  // 256 rows

constexpr int kGemmMaxSmem = 227 * 1024 - 2048;  // dynamic (the static barriers / TMEM slot take the rest)

// Operand chunks travel global -> shared memory with cp.async (16 B, no registers held)
// into a ring of raw fp32 stages several chunks ahead of the tensor core; every thread
// then splits one raw chunk into the hi / lo tf32 tiles the MMAs read.  Raw layouts:
// K-contiguous operands [row][36 floats] (the 4-float pad keeps the split's 16-byte reads
// conflict-free), row-contiguous (transposed) operands [k][R] (the split reads four k of
// one row with scalar loads on distinct banks and stores one 16-byte core-matrix row).
constexpr int kRawRowF = kGemmKc + 4;
// raw chunk bytes: layout T ([k][R], row-contiguous operands) or N ([row][36])
__host__ __device__ constexpr size_t raw_bytes(int r, bool t) { return t ? (size_t)r * kGemmKc * 4 : (size_t)r * kRawRowF * 4; }
__host__ __device__ constexpr size_t split_bytes(int r) { return (size_t)r * kGemmKc * 4 * 2; }  // hi + lo

// Shared-memory plan of one launch: B resident (every K chunk of B split once per CTA -- B
// does not depend on the row tile) when it fits and the CTA has more than one tile.
struct GemmPlan {
    int b_res;
    int raw;  // raw stages (chunks in flight: raw - 1), as many as fit (2 .. kMaxRaw)
    size_t bytes;
};
constexpr int kMaxRaw = 6;  // (cp_async_wait_n covers up to 4 pending groups)
// (one split buffer: measured faster than two with a stage fewer in flight)
inline size_t gemm_bytes(int nt, int nck, bool b_res, bool ta, bool tb, int raw, int nsplit = 1) {
    if (b_res) return (size_t)nck * split_bytes(nt) + raw * raw_bytes(kGemmM, ta) + split_bytes(kGemmM);
    return raw * (raw_bytes(kGemmM, ta) + raw_bytes(nt, tb)) + nsplit * (split_bytes(kGemmM) + split_bytes(nt));
}
// flush: a weight-gradient reduction (two split buffers when B is streamed)
inline GemmPlan gemm_plan(int nt, int nck, bool many_tiles, bool ta, bool tb, bool flush) {
    GemmPlan p{};
    p.b_res = many_tiles && nck > 0 && gemm_bytes(nt, nck, true, ta, tb, 3) <= (size_t)kGemmMaxSmem;
    const int ns = flush && !p.b_res ? 2 : 1;
    p.raw = 2;
    while (p.raw < kMaxRaw && gemm_bytes(nt, nck, p.b_res, ta, tb, p.raw + 1, ns) <= (size_t)kGemmMaxSmem) ++p.raw;
    p.bytes = gemm_bytes(nt, nck, p.b_res, ta, tb, p.raw, ns);
    return p;
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void cp_async_wait_n(int n) {  // n: block-uniform
    switch (n) {
        case 0: cp_async_wait<0>(); break;
        case 1: cp_async_wait<1>(); break;
        case 2: cp_async_wait<2>(); break;
        case 3: cp_async_wait<3>(); break;
        default: cp_async_wait<4>(); break;
    }
}

// 1D bulk copy (TMA engine) global -> shared, completion counted on an mbarrier.
__device__ __forceinline__ void bulk_copy(uint32_t dst, const void* src, uint32_t bytes, uint64_t* mbar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(smem_u32(mbar))
                 : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* mbar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)), "r"(bytes) : "memory");
}

// Mode 2 also takes a partial row tile when every 16-byte run of a k row stays inside the
// row stride (the runs past nrows are read -- they only feed output rows / columns the
// epilogue discards -- or zero-filled).
__device__ __forceinline__ int op_mode(const float* P, int64_t sr, int64_t sk, int r0, int nrows, int k0, int kend,
                                       int R) {
    const bool aligned = ((uintptr_t)P & 15) == 0;
    if (sk == 1 && (sr & 3) == 0 && aligned) return 1;  // (a partial last chunk is zero-filled by cp.async)
    if (sr == 1 && (sk & 3) == 0 && aligned && (r0 & 3) == 0 && (r0 + R <= nrows || (int64_t)((nrows + 3) & ~3) <= sk))
        return 2;
    return 0;
}

// Issue the raw copy of rows [r0, r0 + R) x k [k0, k0 + 32) of X(r, k) = P[r sr + k sk]
// (zeros outside rows < nrows, k < kend); mode 0 copies synchronously.
template <int R, int NTHR = kGemmThreads>
__device__ __forceinline__ void raw_issue(const float* __restrict__ P, int64_t sr, int64_t sk, int r0, int nrows,
                                          int k0, int kend, char* raw) {
    const int mode = op_mode(P, sr, sk, r0, nrows, k0, kend, R);
    const bool lay_t = sr == 1;  // the raw layout (T: [k][R]) follows the operand, not the chunk
    const uint32_t base = smem_u32(raw);
    constexpr int kIt = (R * 8 + NTHR - 1) / NTHR;
    if (mode == 1 && !lay_t) {
#pragma unroll
        for (int it = 0; it < kIt; ++it) {
            const int idx = threadIdx.x + it * NTHR;
            if (R * 8 % NTHR && idx >= R * 8) break;
            const int r = idx >> 3, q = idx & 7, gr = r0 + r;
            const int kv = kend - k0 - 4 * q;  // valid k of this 16-byte run
            const bool ok = gr < nrows && kv > 0;
            cp_async16(base + (uint32_t)(r * kRawRowF * 4 + q * 16), ok ? P + (int64_t)gr * sr + k0 + 4 * q : P,
                       ok ? (uint32_t)min(kv, 4) * 4u : 0u);
        }
    } else if (mode == 2) {  // (implies layout T)
        constexpr int rq_n = R / 4;
#pragma unroll
        for (int it = 0; it < kIt; ++it) {
            const int idx = threadIdx.x + it * NTHR;
            if (R * 8 % NTHR && idx >= R * 8) break;
            const int k = idx / rq_n, rq = idx - k * rq_n, gk = k0 + k;
            const bool ok = gk < kend && r0 + 4 * rq < nrows;
            cp_async16(base + (uint32_t)(k * R * 4 + rq * 16), ok ? P + (r0 + 4 * rq) + (int64_t)gk * sk : P,
                       ok ? 16u : 0u);
        }
    } else {
        float* rf = reinterpret_cast<float*>(raw);
        for (int idx = threadIdx.x; idx < R * kGemmKc; idx += NTHR) {
            const int r = idx / kGemmKc, k = idx - r * kGemmKc, gr = r0 + r, gk = k0 + k;
            rf[lay_t ? k * R + r : r * kRawRowF + k] =
                (gr < nrows && gk < kend) ? P[(int64_t)gr * sr + (int64_t)gk * sk] : 0.f;
        }
    }
}

// Split a raw chunk into the K-major no-swizzle hi / lo tiles (core matrices).
// Layout T rows are ldr floats apart (R, or the operand's own row stride when a bulk copy
// brought the chunk in whole; rows past it then hold other data, which only feeds output
// rows / columns the epilogue discards).
template <int R, int NTHR = kGemmThreads>
__device__ __forceinline__ void raw_split(bool lay_t, const char* raw, char* hi, char* lo, int kvalid = kGemmKc,
                                          float* rsum = nullptr, int ldr = R, int t0 = -1) {
    constexpr int kIt = (R * 8 + NTHR - 1) / NTHR;
    const int tt = t0 < 0 ? (int)threadIdx.x : t0;  // this thread's index among the NTHR splitting
    if (!lay_t) {
#pragma unroll
        for (int it = 0; it < kIt; ++it) {
            const int idx = tt + it * NTHR;
            if (R * 8 % NTHR && idx >= R * 8) break;
            const int r8 = idx & 7, q = (idx >> 3) & 7, rg = idx >> 6, r = rg * 8 + r8;
            const float4 v = *reinterpret_cast<const float4*>(raw + r * kRawRowF * 4 + q * 16);
            float4 h, l;
            split4(v, h, l);
            const uint32_t o = core_off(r, 4 * q);
            *reinterpret_cast<float4*>(hi + o) = h;
            *reinterpret_cast<float4*>(lo + o) = l;
        }
    } else {
        constexpr int rq_n = R / 4;
        const float* rf = reinterpret_cast<const float*>(raw);
#pragma unroll
        for (int it = 0; it < kIt; ++it) {
            const int idx = tt + it * NTHR;
            if (R * 8 % NTHR && idx >= R * 8) break;
            const int kq = idx & 3, rq = (idx >> 2) % rq_n, kb = (idx >> 2) / rq_n, r = 4 * rq + kq;
            float4 v = make_float4(rf[(4 * kb + 0) * ldr + r], rf[(4 * kb + 1) * ldr + r], rf[(4 * kb + 2) * ldr + r],
                                   rf[(4 * kb + 3) * ldr + r]);
            if (4 * kb + 4 > kvalid) {  // rows past a bulk-copied partial chunk hold stale data
                if (4 * kb + 0 >= kvalid) v.x = 0.f;
                if (4 * kb + 1 >= kvalid) v.y = 0.f;
                if (4 * kb + 2 >= kvalid) v.z = 0.f;
                if (4 * kb + 3 >= kvalid) v.w = 0.f;
            }
            float4 h, l;
            split4(v, h, l);
            const uint32_t o = core_off(r, 4 * kb);
            *reinterpret_cast<float4*>(hi + o) = h;
            *reinterpret_cast<float4*>(lo + o) = l;
            if (rsum) rsum[it] += (v.x + v.y) + (v.z + v.w);  // the fused row sum (bias gradient), per group
        }
    }
}

// D[m, n] = sum_k A(m, k) B(n, k) over this CTA's K slice for 128-row tiles (CTAs
// stride over the tiles), n < N (N <= NT).  The chunks of all the CTA's tiles form one
// sequence; chunk q + kRaw - 1 is in flight (cp.async) while chunk q is split and
// multiplied.  Thread 0 issues the 3xTF32 MMAs of a chunk and commits them to mb_mma; the
// split of the next chunk waits for them (one split buffer).  Epilogue per tile: + bias[n],
// ReLU, * (mask(m, n) > 0), store to C + slice * slice_stride (split-K partials are
// reduced by k_reduce_slices).
template <int NT, bool FLUSH, bool BRES>
__global__ void __launch_bounds__(kGemmThreads, 1) k_gemm_tf32x3(GemmArgs g, int kRaw) {
    extern __shared__ __align__(1024) char smem[];
    __shared__ __align__(8) uint64_t mb_mma[2];
    __shared__ __align__(8) uint64_t mb_tile;
    __shared__ __align__(8) uint64_t mb_raw[kMaxRaw];  // bulk mode: raw stage filled
    __shared__ uint32_t tmem_base_s;
    // weight-gradient reductions (FLUSH, both operands streamed): two split buffers (the
    // split of chunk q + 1 overlaps the MMAs of chunk q) and two TMEM accumulators (a
    // group's flush into registers overlaps the next group's MMAs)
    constexpr int kSplit = (FLUSH && !BRES) ? 2 : 1;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr int kAccCols = NT <= 32 ? 32 : (NT <= 64 ? 64 : (NT <= 128 ? 128 : 256));
    constexpr int kTmemCols = FLUSH ? 2 * kAccCols : kAccCols;
    constexpr uint32_t kABytes = kGemmM * kGemmKc * 4, kBBytes = NT * kGemmKc * 4;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)),
                     "n"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        mbar_init(&mb_mma[0], 1);
        mbar_init(&mb_mma[1], 1);
        mbar_init(&mb_tile, 1);
        for (int i = 0; i < kMaxRaw; ++i) mbar_init(&mb_raw[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    const uint32_t tmem = tmem_base_s;
    // TMEM lane quadrant of this warp (warps w, w + 4, ... share it and split the columns
    // into groups of kColHalf >= 16)
    const uint32_t tl = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    constexpr int kEpiGroups = NT >= 64 ? 4 : (NT == 32 ? 2 : 1);
    constexpr int kColHalf = NT / kEpiGroups;
    const int col0 = ((warp >> 2) % kEpiGroups) * kColHalf;
    const bool epi_warp = (warp >> 2) < kEpiGroups;

    const int slice = blockIdx.y;
    const int kbeg = slice * g.k_per_slice;
    const int kend = min(g.K, kbeg + g.k_per_slice);
    const int ntiles = (g.M + kGemmM - 1) / kGemmM;
    const int nck = kend > kbeg ? (kend - kbeg + kGemmKc - 1) / kGemmKc : 0;
    const int my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    constexpr uint32_t idesc = idesc_tf32(kGemmM, NT);
    float* C = g.C + (int64_t)slice * g.slice_stride;
    // shared memory: [B split chunks (resident)] [split buffers: A hi, A lo (, B hi, B lo)] [raw stages: A (, B)]
    const bool ta = g.a_m == 1, tb = g.b_n == 1;  // raw layouts
    char* bres = smem;
    char* split0 = smem + (BRES ? (size_t)nck * 2 * kBBytes : 0);
    constexpr size_t kSplitBuf = BRES ? 2 * kABytes : 2 * kABytes + 2 * kBBytes;
    char* raw0 = split0 + kSplit * kSplitBuf;
    const size_t raw_sa = raw_bytes(kGemmM, ta), raw_stage = raw_sa + (BRES ? 0 : raw_bytes(NT, tb));
    auto raw_a = [&](int st) { return raw0 + (size_t)st * raw_stage; };
    auto raw_b = [&](int st) { return raw0 + (size_t)st * raw_stage + raw_sa; };
    if (BRES) {  // B split once: through raw stage 0
        for (int ch = 0; ch < nck; ++ch) {
            const int k0 = kbeg + ch * kGemmKc;
            raw_issue<NT>(g.B, g.b_n, g.b_k, 0, g.N, k0, kend, raw_a(0));  // (raw A stage 0 as scratch)
            cp_async_commit();
            cp_async_wait<0>();
            __syncthreads();
            char* bh = bres + (size_t)ch * 2 * kBBytes;
            raw_split<NT>(tb, raw_a(0), bh, bh + kBBytes);
            __syncthreads();
        }
    }
    const int total = my_tiles * nck;
    // Bulk mode (both operands row-contiguous with one tile each: M <= row stride <= 128,
    // N <= row stride <= NT, so a chunk of each is one contiguous run of 32 rows): one TMA
    // bulk copy per operand per chunk, completion on the stage's mbarrier, the whole ring in
    // flight.  Otherwise per-thread cp.async.
    const bool bulk = !BRES && ta && tb && g.M <= g.a_k && g.a_k <= kGemmM && g.N <= g.b_k && g.b_k <= NT &&
                      ((g.a_k | g.b_k) & 3) == 0 && (((uintptr_t)g.A | (uintptr_t)g.B) & 15) == 0;
    const int lda = bulk ? (int)g.a_k : kGemmM, ldb = bulk ? (int)g.b_k : NT;  // raw T row strides
    // issue cursor: the next chunk to load (tile row m0, chunk ch, raw stage)
    int is_q = 0, is_m0 = (int)blockIdx.x * kGemmM, is_ch = 0, is_st = 0;
    auto issue_bulk = [&]() {  // thread 0: the next chunk (nothing past the end)
        if (is_q < total) {
            const int k0 = kbeg + is_ch * kGemmKc, rows = min(kGemmKc, kend - k0);
            const uint32_t ba = (uint32_t)rows * lda * 4, bb = (uint32_t)rows * ldb * 4;
            mbar_expect_tx(&mb_raw[is_st], ba + bb);
            bulk_copy(smem_u32(raw_a(is_st)), g.A + (int64_t)k0 * lda, ba, &mb_raw[is_st]);
            bulk_copy(smem_u32(raw_b(is_st)), g.B + (int64_t)k0 * ldb, bb, &mb_raw[is_st]);
            if (++is_ch == nck) {
                is_ch = 0;
                is_m0 += (int)gridDim.x * kGemmM;
            }
            if (++is_st == kRaw) is_st = 0;
            ++is_q;
        }
    };
    auto issue = [&]() {  // the next chunk of the sequence (an empty group past the end)
        if (is_q < total) {
            const int k0 = kbeg + is_ch * kGemmKc;
            raw_issue<kGemmM>(g.A, g.a_m, g.a_k, is_m0, g.M, k0, kend, raw_a(is_st));
            if (!BRES) raw_issue<NT>(g.B, g.b_n, g.b_k, 0, g.N, k0, kend, raw_b(is_st));
            if (++is_ch == nck) {
                is_ch = 0;
                is_m0 += (int)gridDim.x * kGemmM;
            }
            if (++is_st == kRaw) is_st = 0;
            ++is_q;
        }
        cp_async_commit();
    };
    if (bulk) {
        if (tid == 0)
            for (int q = 0; q < kRaw; ++q) issue_bulk();
    } else {
        for (int q = 0; q < kRaw - 1; ++q) issue();
    }
    int rd_st = 0;         // raw stage of chunk q
    uint32_t rd_ph = 0;    // its fill parity (bulk mode)
    // fused row sums of A (the bias gradient of a weight-gradient GEMM): per thread its rows
    constexpr int kRsIt = (kGemmM * 8 + kGemmThreads - 1) / kGemmThreads;
    // (fp32 within an accumulation group of kFlushChunks chunks, folded into fp64 per group:
    // an fp64 add chain per chunk stalled the split)
    double rsum[kRsIt];
    float rsf[kRsIt];
#pragma unroll
    for (int i = 0; i < kRsIt; ++i) {
        rsum[i] = 0.0;
        rsf[i] = 0.f;
    }
    const bool do_rsum = g.rowsum && ta && !BRES;
    uint32_t tphase = 0;  // mb_tile completions waited for
    float acc[FLUSH ? kColHalf : 1];
    int G = -1;  // running accumulation group (FLUSH: its accumulator is G & 1)
    auto flush = [&](int grp) {  // add group grp's accumulator (MMAs committed to mb_tile) into acc
        mbar_wait(&mb_tile, tphase & 1u);
        ++tphase;
        tc_after_sync();
#pragma unroll
        for (int cc = 0; cc < kColHalf; cc += 16) {
            uint32_t v[16];
            tmem_ld16(tl + (uint32_t)((grp & 1) * kAccCols + col0 + cc), v);
#pragma unroll
            for (int j = 0; j < 16; ++j) acc[(FLUSH ? cc : 0) + j] += __uint_as_float(v[j]);
        }
        tc_before_sync();  // the group after next overwrites this accumulator
    };
    for (int t = 0, q = 0; t < my_tiles; ++t) {
        const int m0 = ((int)blockIdx.x + t * (int)gridDim.x) * kGemmM;
#pragma unroll
        for (int j = 0; j < (FLUSH ? kColHalf : 1); ++j) acc[j] = 0.f;
        for (int chunk = 0; chunk < nck; ++chunk, ++q) {
            const int k0 = kbeg + chunk * kGemmKc;
            if (bulk) {
                mbar_wait(&mb_raw[rd_st], rd_ph);  // chunk q landed
            } else {
                cp_async_wait_n(kRaw - 2);  // chunk q landed (this thread's copies)
                __syncthreads();            // ... everyone's; raw stage (q - 1) % kRaw is free again
                issue();
            }
            // the split buffer's previous MMAs (chunk q - kSplit) are done
            if (q >= kSplit) mbar_wait(&mb_mma[q % kSplit], (uint32_t)(q / kSplit - 1) & 1u);
            tc_after_sync();
            char* a_hi = split0 + (size_t)(q % kSplit) * kSplitBuf;
            char* a_lo = a_hi + kABytes;
            char* sb_hi = a_lo + kABytes;  // split B (not resident)
            const int kvalid = bulk ? min(kGemmKc, kend - k0) : kGemmKc;
            raw_split<kGemmM>(ta, raw_a(rd_st), a_hi, a_lo, kvalid, do_rsum ? rsf : nullptr, lda);
            if (!BRES) raw_split<NT>(tb, raw_b(rd_st), sb_hi, sb_hi + kBBytes, kvalid, nullptr, ldb);
            if (++rd_st == kRaw) {
                rd_st = 0;
                rd_ph ^= 1u;
            }
            fence_async_smem();
            __syncthreads();
            if (bulk && tid == 0) issue_bulk();  // into the stage just split (chunk q + kRaw)
            const bool group_start = FLUSH ? (chunk % kFlushChunks) == 0 : chunk == 0;
            const bool group_end = FLUSH ? ((chunk % kFlushChunks) == kFlushChunks - 1 || chunk + 1 == nck)
                                         : chunk + 1 == nck;
            if (group_start) ++G;
            if (do_rsum && group_end) {
#pragma unroll
                for (int i = 0; i < kRsIt; ++i) {
                    rsum[i] += (double)rsf[i];
                    rsf[i] = 0.f;
                }
            }
            const uint32_t dacc = tmem + (uint32_t)(FLUSH ? (G & 1) * kAccCols : 0);
            // the previous group's flush runs after this chunk's MMAs are issued, except when this
            // chunk alone is a group: its end commit could then complete mb_tile a second time
            // before the flush waited for the first (a parity wait cannot tell them apart)
            const bool flush_now = FLUSH && group_start && chunk > 0, flush_first = flush_now && group_end;
            if (flush_first) flush(G - 1);
            if (tid == 0) {
                tc_after_sync();
                char* b_hi = BRES ? bres + (size_t)chunk * 2 * kBBytes : sb_hi;
                char* b_lo = b_hi + kBBytes;
                const uint32_t ah = smem_u32(a_hi), al = smem_u32(a_lo), bh = smem_u32(b_hi), bl = smem_u32(b_lo);
#pragma unroll
                for (int s = 0; s < kGemmKc / 8; ++s) {  // K = 8 tf32 per MMA = 2 core-matrix columns
                    const uint32_t off = (uint32_t)s * 2u * kCoreBytes;
                    const uint64_t dah = umma_desc(ah + off, kCoreBytes, kGroupBytes);
                    const uint64_t dal = umma_desc(al + off, kCoreBytes, kGroupBytes);
                    const uint64_t dbh = umma_desc(bh + off, kCoreBytes, kGroupBytes);
                    const uint64_t dbl = umma_desc(bl + off, kCoreBytes, kGroupBytes);
                    mma_tf32(dacc, dah, dbh, idesc, (!group_start || s > 0) ? 1u : 0u);
                    mma_tf32(dacc, dah, dbl, idesc, 1u);
                    mma_tf32(dacc, dal, dbh, idesc, 1u);
                }
                mma_commit(&mb_mma[q % kSplit]);
                if (group_end) mma_commit(&mb_tile);
            }
            // the previous group's flush, while this group's first MMAs run
            if (flush_now && !flush_first) flush(G - 1);
        }
        if (FLUSH && nck > 0) flush(G);  // the tile's last group
        const bool any = nck > 0;
        // the epilogue's mask loads go out before the wait for the tile's last MMAs
        const int m = m0 + (warp & 3) * 32 + lane;
        const bool row_ok = m < g.M;
        const float* mrow0 = g.mask && row_ok && epi_warp ? g.mask + (int64_t)m * g.ldmask + col0 : nullptr;
        const bool mvec = mrow0 && ((uintptr_t)mrow0 & 15) == 0 && (g.ldmask & 3) == 0;
        float4 mk[kColHalf / 4];
        uint32_t mbits = 0xffffffffu;  // gate bits of columns col0 .. col0 + 31 (bit gates)
        if (g.maskbits && row_ok && epi_warp) mbits = __ldg(g.maskbits + (int64_t)m * g.ldmaskbits + (col0 >> 5));
        mbits >>= col0 & 31;
#pragma unroll
        for (int i = 0; i < kColHalf / 4; ++i)
            mk[i] = mvec && col0 + 4 * i + 4 <= g.N ? __ldg(reinterpret_cast<const float4*>(mrow0) + i)
                                                  : make_float4(1.f, 1.f, 1.f, 1.f);
        if (!FLUSH && any) {
            mbar_wait(&mb_tile, tphase & 1u);
            ++tphase;
            tc_after_sync();
        }

        // epilogue: this warp's TMEM lane quadrant (rows), its column group.  The mask loads
        // of the whole group are issued before any store (C may alias nothing, but the
        // compiler cannot know it: load / store pairs would serialise on memory latency).
        if (epi_warp) {
#pragma unroll
            for (int cc = 0; cc < kColHalf; cc += 16) {
                const int n0 = col0 + cc;
                uint32_t v[16];
                if (FLUSH) {
#pragma unroll
                    for (int j = 0; j < 16; ++j) v[j] = __float_as_uint(acc[(FLUSH ? cc : 0) + j]);
                } else if (any) {
                    tmem_ld16(tl + (uint32_t)n0, v);
                } else {
#pragma unroll
                    for (int j = 0; j < 16; ++j) v[j] = 0u;
                }
                if (row_ok && n0 < g.N) {
                    float x[16];
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        x[j] = __uint_as_float(v[j]);
                        if (g.bias && n0 + j < g.N) x[j] += __ldg(g.bias + n0 + j);
                        if (g.relu) x[j] = fmaxf(x[j], 0.f);
                        if (!((mbits >> (cc + j)) & 1u)) x[j] = 0.f;
                    }
                    float* crow = C + (int64_t)m * g.ldc + n0;
                    const float* mrow = g.mask ? g.mask + (int64_t)m * g.ldmask + n0 : nullptr;
                    const bool vec = n0 + 16 <= g.N && ((uintptr_t)crow & 15) == 0 && (!mrow || mvec);
                    if (vec) {
#pragma unroll
                        for (int q4 = 0; q4 < 4; ++q4) {
                            const float4 mq = mk[cc / 4 + q4];
                            float4 o = make_float4(x[4 * q4], x[4 * q4 + 1], x[4 * q4 + 2], x[4 * q4 + 3]);
                            if (!(mq.x > 0.f)) o.x = 0.f;
                            if (!(mq.y > 0.f)) o.y = 0.f;
                            if (!(mq.z > 0.f)) o.z = 0.f;
                            if (!(mq.w > 0.f)) o.w = 0.f;
                            reinterpret_cast<float4*>(crow)[q4] = o;
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            if (n0 + j >= g.N) break;
                            float xv = x[j];
                            if (mrow && !(mrow[j] > 0.f)) xv = 0.f;
                            crow[j] = xv;
                        }
                    }
                }
            }
        }
        tc_before_sync();  // the next tile's first MMA overwrites the accumulator
    }
    cp_async_wait<0>();
    tc_before_sync();
    __syncthreads();
    if (do_rsum) {  // per row: the partials of the threads that split its k groups, in a fixed order
        double* red = reinterpret_cast<double*>(raw0);  // [k group][row] (the ring is idle now)
        constexpr int rq_n = kGemmM / 4;
#pragma unroll
        for (int it = 0; it < kRsIt; ++it) {
            const int idx = threadIdx.x + it * kGemmThreads;
            if (idx >= kGemmM * 8) break;
            const int kq = idx & 3, rq = (idx >> 2) % rq_n, kb = (idx >> 2) / rq_n;
            red[kb * kGemmM + 4 * rq + kq] = rsum[it];
        }
        __syncthreads();
        if (tid < g.M) {
            double t = 0.0;
            for (int kb = 0; kb < kGemmKc / 4; ++kb) t += red[kb * kGemmM + tid];
            g.rowsum[(int64_t)slice * g.M + tid] = (float)t;
        }
    }
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols) : "memory");
}

// sin / cos (pi 2^l v) for l = 0, 1, ...: one fp64 sincospi, then the double-angle step
// (sin 2x = 2 s c, cos 2x = (c - s)(c + s)) per level -- the fp64 error doubles per level
// (~1e-13 at level 9), far below the fp32 rounding of the encoding.
__device__ __forceinline__ void sincospi_double(double& s, double& c) {
    const double s2 = 2.0 * s * c;
    c = (c - s) * (c + s);
    s = s2;
}

__device__ __forceinline__ void tmem_ld16_nw(uint32_t taddr, uint32_t* v) {  // (no wait: tmem_wait_ld)
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// 256-bit global store (sm_100): one whole 32-byte sector per thread
__device__ __forceinline__ void st_v8(float* p, const float* x) {
    asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "f"(x[0]), "f"(x[1]), "f"(x[2]),
                 "f"(x[3]), "f"(x[4]), "f"(x[5]), "f"(x[6]), "f"(x[7])
                 : "memory");
}

__device__ __forceinline__ float* C_row(const GemmArgs& g, int m) { return g.C + (int64_t)m * g.ldc; }

// Warp-specialised variant for resident-B GEMMs without split-K (the input gradients
// delta W and the layer-by-layer forward): warps 0-7 load (cp.async ring), split and issue
// the MMAs (thread 0); warps 8-15 drain the finished tile's accumulator (bias, ReLU, gate,
// stores).  Two TMEM accumulators alternate between tiles, so a tile's epilogue runs while
// the next tile's chunks are loaded, split and multiplied (acc_full: MMAs of the tile done;
// acc_empty: its epilogue has read the accumulator).
__device__ __forceinline__ void bar_main() { asm volatile("bar.sync 1, %0;" ::"n"(kGemmThreads / 2) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* mbar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(mbar)) : "memory");
}

constexpr int kEpiLd = 20;  // staging row stride (floats): 16 columns + 4 (conflict-free float4 rows)
constexpr size_t kEpiStageBytes = (size_t)(kGemmThreads / 64) * 32 * kEpiLd * 4;  // 8 epilogue warps

template <int NT>
__global__ void __launch_bounds__(kGemmThreads, 1) k_gemm_ws(GemmArgs g, int kRaw) {
    extern __shared__ __align__(1024) char smem[];
    __shared__ __align__(8) uint64_t mb_mma, acc_full[2], acc_empty[2];
    __shared__ uint32_t tmem_base_s;
    constexpr int kMain = kGemmThreads / 2;
    constexpr int kEpiWarps = (kGemmThreads - kMain) / 32;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr int kAccCols = NT <= 32 ? 32 : (NT <= 64 ? 64 : 128);
    constexpr int kTmemCols = 2 * kAccCols;
    constexpr uint32_t kABytes = kGemmM * kGemmKc * 4, kBBytes = NT * kGemmKc * 4;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)),
                     "n"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        mbar_init(&mb_mma, 1);
        for (int b = 0; b < 2; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], kEpiWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    const uint32_t tmem = tmem_base_s;
    const int kend = g.K;
    const int ntiles = (g.M + kGemmM - 1) / kGemmM;
    const int nck = (kend + kGemmKc - 1) / kGemmKc;  // (> 0: the launcher routes K = 0 elsewhere)
    const int my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    constexpr uint32_t idesc = idesc_tf32(kGemmM, NT);
    const bool ta = g.a_m == 1, tb = g.b_n == 1;
    char* bres = smem;
    char* split0 = smem + (size_t)nck * 2 * kBBytes;
    char* raw0 = split0 + 2 * kABytes;
    const size_t raw_stage = raw_bytes(kGemmM, ta);
    auto raw_a = [&](int st) { return raw0 + (size_t)st * raw_stage; };
    for (int ch = 0; ch < nck; ++ch) {  // B split once by all warps, through raw stage 0
        const int k0 = ch * kGemmKc;
        raw_issue<NT>(g.B, g.b_n, g.b_k, 0, g.N, k0, kend, raw_a(0));
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
        char* bh = bres + (size_t)ch * 2 * kBBytes;
        raw_split<NT>(tb, raw_a(0), bh, bh + kBBytes);
        __syncthreads();
    }
    if (warp < kMain / 32) {
        // ---- loads, split, MMAs ----
        const int total = my_tiles * nck;
        int is_q = 0, is_m0 = (int)blockIdx.x * kGemmM, is_ch = 0, is_st = 0;
        auto issue = [&]() {
            if (is_q < total) {
                raw_issue<kGemmM, kMain>(g.A, g.a_m, g.a_k, is_m0, g.M, is_ch * kGemmKc, kend, raw_a(is_st));
                if (++is_ch == nck) {
                    is_ch = 0;
                    is_m0 += (int)gridDim.x * kGemmM;
                }
                if (++is_st == kRaw) is_st = 0;
                ++is_q;
            }
            cp_async_commit();
        };
        for (int q = 0; q < kRaw - 1; ++q) issue();
        int rd_st = 0;
        char* a_hi = split0;
        char* a_lo = split0 + kABytes;
        for (int t = 0, q = 0; t < my_tiles; ++t) {
            const int buf = t & 1;
            for (int chunk = 0; chunk < nck; ++chunk, ++q) {
                cp_async_wait_n(kRaw - 2);  // chunk q landed (this thread's copies)
                bar_main();                 // ... everyone's; raw stage (q - 1) % kRaw is free again
                issue();
                if (q >= 1) mbar_wait(&mb_mma, (uint32_t)(q - 1) & 1u);  // the split buffer's MMAs are done
                tc_after_sync();
                raw_split<kGemmM, kMain>(ta, raw_a(rd_st), a_hi, a_lo);
                if (++rd_st == kRaw) rd_st = 0;
                fence_async_smem();
                bar_main();
                if (tid == 0) {
                    if (chunk == 0 && t >= 2) mbar_wait(&acc_empty[buf], (uint32_t)((t >> 1) - 1) & 1u);
                    tc_after_sync();
                    const uint32_t d = tmem + (uint32_t)(buf * kAccCols);
                    const char* b_hi = bres + (size_t)chunk * 2 * kBBytes;
                    const uint32_t ah = smem_u32(a_hi), al = smem_u32(a_lo), bh = smem_u32(b_hi),
                                   bl = smem_u32(b_hi + kBBytes);
#pragma unroll
                    for (int s = 0; s < kGemmKc / 8; ++s) {
                        const uint32_t off = (uint32_t)s * 2u * kCoreBytes;
                        const uint64_t dah = umma_desc(ah + off, kCoreBytes, kGroupBytes);
                        const uint64_t dal = umma_desc(al + off, kCoreBytes, kGroupBytes);
                        const uint64_t dbh = umma_desc(bh + off, kCoreBytes, kGroupBytes);
                        const uint64_t dbl = umma_desc(bl + off, kCoreBytes, kGroupBytes);
                        mma_tf32(d, dah, dbh, idesc, (chunk > 0 || s > 0) ? 1u : 0u);
                        mma_tf32(d, dah, dbl, idesc, 1u);
                        mma_tf32(d, dal, dbh, idesc, 1u);
                    }
                    mma_commit(&mb_mma);
                    if (chunk + 1 == nck) mma_commit(&acc_full[buf]);
                }
            }
        }
        cp_async_wait<0>();
    } else {
        // ---- epilogue: TMEM lane quadrant warp % 4, column half (warp - 8) / 4 ----
        const int ew = warp - kMain / 32;
        const uint32_t tl = tmem + ((uint32_t)((warp & 3) * 32) << 16);
        // warp-private staging blocks after the raw ring (kEpiStageBytes, reserved by the launcher)
        float* epi_stage = reinterpret_cast<float*>(raw0 + (size_t)kRaw * raw_stage);
        const bool staged = !g.mask && (g.N & 3) == 0 && (g.ldc & 3) == 0 && (((uintptr_t)g.C) & 15) == 0;
        constexpr int kEpiGroups = NT >= 32 ? 2 : 1;
        constexpr int kColHalf = NT / kEpiGroups;
        const int col0 = ((ew >> 2) % kEpiGroups) * kColHalf;
        const bool epi_warp = (ew >> 2) < kEpiGroups;
        for (int t = 0; t < my_tiles; ++t) {
            const int buf = t & 1;
            const int m0 = ((int)blockIdx.x + t * (int)gridDim.x) * kGemmM;
            const int m = m0 + (warp & 3) * 32 + lane;
            const bool row_ok = m < g.M;
            // the gate loads go out before the wait for the tile's MMAs
            const float* mrow0 = g.mask && row_ok && epi_warp ? g.mask + (int64_t)m * g.ldmask + col0 : nullptr;
            const bool mvec = mrow0 && ((uintptr_t)mrow0 & 15) == 0 && (g.ldmask & 3) == 0;
            uint32_t mb0 = 0xffffffffu, mb1 = 0xffffffffu;  // gate bit words of the column group
            if (g.maskbits && row_ok && epi_warp) {
                const uint32_t* pb = g.maskbits + (int64_t)m * g.ldmaskbits + (col0 >> 5);
                mb0 = __ldg(pb);
                if (((col0 + kColHalf - 1) >> 5) > (col0 >> 5)) mb1 = __ldg(pb + 1);
            }
            mbar_wait(&acc_full[buf], (uint32_t)(t >> 1) & 1u);
            tc_after_sync();
            // the whole column group out of TMEM first (one wait), then the accumulator is
            // released for the tile after next before any store is issued
            uint32_t v[kColHalf];
            if (epi_warp) {
#pragma unroll
                for (int cc = 0; cc < kColHalf; cc += 16) tmem_ld16_nw(tl + (uint32_t)(buf * kAccCols + col0 + cc), v + cc);
                tmem_wait_ld();
            }
            tc_before_sync();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[buf]);
            if (NT == 128 && g.chain_x) {  // fused encoding chain (column group 0 holds the 63 x columns)
                if (epi_warp && row_ok && col0 == 0) {
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const double xv = (double)__ldg(g.chain_x + (int64_t)m * g.chain_ldx + 21 * c);
                        double acc = (double)__uint_as_float(v[21 * c]);
                        double fr = M_PI, sn, cs;
                        sincospi(xv, &sn, &cs);
#pragma unroll
                        for (int l = 0; l < 10; ++l, fr *= 2.0) {
                            if (l) sincospi_double(sn, cs);
                            acc += fr * cs * (double)__uint_as_float(v[21 * c + 1 + 2 * l]) -
                                   fr * sn * (double)__uint_as_float(v[21 * c + 2 + 2 * l]);
                        }
                        float* o = g.chain_dpos + (int64_t)m * g.chain_pstride + c;
                        const float val = (float)(acc * g.chain_inv_scale);
                        *o = g.chain_acc ? *o + val : val;
                    }
                }
            } else if (epi_warp && staged) {
                // row-major stores through a warp-private staging block: the TMEM read-out
                // gives a lane one row's 16 columns (a warp store would touch 32 rows / cache
                // lines); after the transpose a warp store writes 8 rows x 64 contiguous bytes
                float* stg = epi_stage + (size_t)(warp - kMain / 32) * 32 * kEpiLd;
                const int rr = lane >> 2, qq = lane & 3;
#pragma unroll
                for (int cc = 0; cc < kColHalf; cc += 16) {
                    const int n0 = col0 + cc;
                    if (n0 >= g.N) continue;
                    const uint32_t bits = ((n0 >> 5) > (col0 >> 5) ? mb1 : mb0) >> (n0 & 31);
                    float x[16];
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        x[j] = __uint_as_float(v[cc + j]);
                        if (g.bias && n0 + j < g.N) x[j] += __ldg(g.bias + n0 + j);
                        if (g.relu) x[j] = fmaxf(x[j], 0.f);
                        if (!((bits >> j) & 1u)) x[j] = 0.f;
                    }
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4)
                        *reinterpret_cast<float4*>(stg + lane * kEpiLd + 4 * q4) =
                            make_float4(x[4 * q4], x[4 * q4 + 1], x[4 * q4 + 2], x[4 * q4 + 3]);
                    __syncwarp();
                    const bool colv = n0 + 4 * qq + 4 <= g.N;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int row = 8 * j + rr;
                        const int mm = m0 + (warp & 3) * 32 + row;
                        const float4 o = *reinterpret_cast<const float4*>(stg + row * kEpiLd + 4 * qq);
                        if (mm < g.M && colv) *reinterpret_cast<float4*>(C_row(g, mm) + n0 + 4 * qq) = o;
                    }
                    __syncwarp();
                }
            } else if (epi_warp && row_ok) {
#pragma unroll
                for (int cc = 0; cc < kColHalf; cc += 16) {
                    const int n0 = col0 + cc;
                    if (n0 >= g.N) continue;
                    const uint32_t bits = ((n0 >> 5) > (col0 >> 5) ? mb1 : mb0) >> (n0 & 31);
                    float x[16];
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        x[j] = __uint_as_float(v[cc + j]);
                        if (g.bias && n0 + j < g.N) x[j] += __ldg(g.bias + n0 + j);
                        if (g.relu) x[j] = fmaxf(x[j], 0.f);
                        if (!((bits >> j) & 1u)) x[j] = 0.f;
                    }
                    float* crow = C_row(g, m) + n0;
                    const float* mrow = mrow0 ? mrow0 + cc : nullptr;
                    if (n0 + 16 <= g.N && !mrow && ((uintptr_t)crow & 31) == 0) {
                        st_v8(crow, x);  // 32-byte stores: whole sectors per lane
                        st_v8(crow + 8, x + 8);
                    } else if (n0 + 16 <= g.N && ((uintptr_t)crow & 15) == 0 && (!mrow || mvec)) {
#pragma unroll
                        for (int q4 = 0; q4 < 4; ++q4) {
                            float4 o = make_float4(x[4 * q4], x[4 * q4 + 1], x[4 * q4 + 2], x[4 * q4 + 3]);
                            if (mrow) {
                                const float4 mq = __ldg(reinterpret_cast<const float4*>(mrow) + q4);
                                if (!(mq.x > 0.f)) o.x = 0.f;
                                if (!(mq.y > 0.f)) o.y = 0.f;
                                if (!(mq.z > 0.f)) o.z = 0.f;
                                if (!(mq.w > 0.f)) o.w = 0.f;
                            }
                            reinterpret_cast<float4*>(crow)[q4] = o;
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < 16; ++j)
                            if (n0 + j < g.N) crow[j] = (mrow && !(mrow[j] > 0.f)) ? 0.f : x[j];
                    }
                }
            }
        }
    }
    tc_before_sync();
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols) : "memory");
}

// Weight-gradient reduction (FLUSH) over one row tile with both operands bulk-copied,
// warp-specialised: warp 0 issues the bulk copies and the MMAs (thread 0), warps 1-15 split;
// every warp flushes its share of the accumulators.  Nothing is block-synchronous inside the
// K loop:
//   mb_raw[st]     a raw stage landed (TMA complete_tx)
//   split_full[b]  the 15 split warps have split chunk q (b = q & 1) -> MMAs; its raw stage
//                  is refilled with chunk q + kRaw
//   mb_mma[b]      chunk q's MMAs done -> split buffer b may take chunk q + 2
//   mb_tile        an accumulation group's MMAs done -> flush (each warp its share)
//   acc_free[a]    all 16 warps flushed accumulator a -> the group after next may use it
template <int NT>
__global__ void __launch_bounds__(kGemmThreads, 1) k_gemm_wsf(GemmArgs g, int kRaw) {
    extern __shared__ __align__(1024) char smem[];
    __shared__ __align__(8) uint64_t mb_raw[kMaxRaw], split_full[2], mb_mma[2], mb_tile, acc_free[2];
    __shared__ uint32_t tmem_base_s;
    constexpr int kSplitThr = kGemmThreads - 32;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr int kAccCols = NT <= 32 ? 32 : (NT <= 64 ? 64 : 128);
    constexpr int kTmemCols = 2 * kAccCols;
    constexpr uint32_t kABytes = kGemmM * kGemmKc * 4, kBBytes = NT * kGemmKc * 4;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)),
                     "n"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        for (int i = 0; i < kMaxRaw; ++i) mbar_init(&mb_raw[i], 1);
        for (int b = 0; b < 2; ++b) {
            mbar_init(&split_full[b], kSplitThr / 32);
            mbar_init(&mb_mma[b], 1);
            mbar_init(&acc_free[b], kGemmThreads / 32);
        }
        mbar_init(&mb_tile, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    const uint32_t tmem = tmem_base_s;
    const uint32_t tl = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    constexpr int kEpiGroups = NT >= 64 ? 4 : (NT == 32 ? 2 : 1);
    constexpr int kColHalf = NT / kEpiGroups;
    const int col0 = ((warp >> 2) % kEpiGroups) * kColHalf;
    const bool epi_warp = (warp >> 2) < kEpiGroups;
    const int slice = blockIdx.y;
    const int kbeg = slice * g.k_per_slice;
    const int kend = min(g.K, kbeg + g.k_per_slice);
    const int nck = kend > kbeg ? (kend - kbeg + kGemmKc - 1) / kGemmKc : 0;
    constexpr uint32_t idesc = idesc_tf32(kGemmM, NT);
    const int lda = (int)g.a_k, ldb = (int)g.b_k;
    char* split0 = smem;
    constexpr size_t kSplitBuf = 2 * kABytes + 2 * kBBytes;
    char* raw0 = split0 + 2 * kSplitBuf;
    const size_t raw_sa = raw_bytes(kGemmM, true), raw_stage = raw_sa + raw_bytes(NT, true);
    auto raw_a = [&](int st) { return raw0 + (size_t)st * raw_stage; };
    auto raw_b = [&](int st) { return raw0 + (size_t)st * raw_stage + raw_sa; };
    auto issue_bulk = [&](int q) {  // thread 0: chunk q into raw stage q % kRaw
        const int k0 = kbeg + q * kGemmKc, rows = min(kGemmKc, kend - k0), st = q % kRaw;
        const uint32_t ba = (uint32_t)rows * lda * 4, bb = (uint32_t)rows * ldb * 4;
        mbar_expect_tx(&mb_raw[st], ba + bb);
        bulk_copy(smem_u32(raw_a(st)), g.A + (int64_t)k0 * lda, ba, &mb_raw[st]);
        bulk_copy(smem_u32(raw_b(st)), g.B + (int64_t)k0 * ldb, bb, &mb_raw[st]);
    };
    float acc[kColHalf];
#pragma unroll
    for (int j = 0; j < kColHalf; ++j) acc[j] = 0.f;
    uint32_t tphase = 0;
    auto flush = [&](int grp) {
        mbar_wait(&mb_tile, tphase & 1u);
        ++tphase;
        tc_after_sync();
        if (epi_warp) {
#pragma unroll
            for (int cc = 0; cc < kColHalf; cc += 16) {
                uint32_t v[16];
                tmem_ld16(tl + (uint32_t)((grp & 1) * kAccCols + col0 + cc), v);
#pragma unroll
                for (int j = 0; j < 16; ++j) acc[cc + j] += __uint_as_float(v[j]);
            }
        }
        tc_before_sync();
    };
    constexpr int kRsIt = (kGemmM * 8 + kSplitThr - 1) / kSplitThr;
    double rsum[kRsIt];
    float rsf[kRsIt];
#pragma unroll
    for (int i = 0; i < kRsIt; ++i) {
        rsum[i] = 0.0;
        rsf[i] = 0.f;
    }
    const bool do_rsum = g.rowsum != nullptr;
    int G = -1;
    if (warp == 0) {
        // ---- bulk copies + MMAs ----
        if (lane == 0)
            for (int q = 0; q < min(kRaw, nck); ++q) issue_bulk(q);
        for (int q = 0; q < nck; ++q) {
            const bool group_start = (q % kFlushChunks) == 0;
            const bool group_end = (q % kFlushChunks) == kFlushChunks - 1 || q + 1 == nck;
            if (group_start) ++G;
            // the previous group's flush: after this chunk's MMAs are issued, except when this
            // chunk alone is a group (its end commit would complete mb_tile a second time
            // before this warp waited for the first: a parity wait cannot tell them apart)
            const bool flush_now = group_start && q > 0, flush_first = flush_now && group_end;
            if (flush_first) {
                flush(G - 1);
                __syncwarp();
                if (lane == 0) mbar_arrive(&acc_free[(G - 1) & 1]);
            }
            if (lane == 0) {
                mbar_wait(&split_full[q & 1], (uint32_t)(q >> 1) & 1u);
                if (group_start && G >= 2) mbar_wait(&acc_free[G & 1], (uint32_t)((G >> 1) - 1) & 1u);
                tc_after_sync();
                const uint32_t dacc = tmem + (uint32_t)((G & 1) * kAccCols);
                const char* a_hi = split0 + (size_t)(q & 1) * kSplitBuf;
                const uint32_t ah = smem_u32(a_hi), al = ah + kABytes, bh = al + kABytes, bl = bh + kBBytes;
#pragma unroll
                for (int s = 0; s < kGemmKc / 8; ++s) {
                    const uint32_t off = (uint32_t)s * 2u * kCoreBytes;
                    const uint64_t dah = umma_desc(ah + off, kCoreBytes, kGroupBytes);
                    const uint64_t dal = umma_desc(al + off, kCoreBytes, kGroupBytes);
                    const uint64_t dbh = umma_desc(bh + off, kCoreBytes, kGroupBytes);
                    const uint64_t dbl = umma_desc(bl + off, kCoreBytes, kGroupBytes);
                    mma_tf32(dacc, dah, dbh, idesc, (!group_start || s > 0) ? 1u : 0u);
                    mma_tf32(dacc, dah, dbl, idesc, 1u);
                    mma_tf32(dacc, dal, dbh, idesc, 1u);
                }
                mma_commit(&mb_mma[q & 1]);
                if (group_end) mma_commit(&mb_tile);
                if (q + kRaw < nck) issue_bulk(q + kRaw);  // chunk q's raw stage has been split
            }
            __syncwarp();
            if (flush_now && !flush_first) {
                flush(G - 1);
                __syncwarp();
                if (lane == 0) mbar_arrive(&acc_free[(G - 1) & 1]);
            }
        }
    } else {
        // ---- split ----
        const int t = tid - 32;
        for (int q = 0; q < nck; ++q) {
            const bool group_start = (q % kFlushChunks) == 0;
            const bool group_end = (q % kFlushChunks) == kFlushChunks - 1 || q + 1 == nck;
            if (group_start) ++G;
            const bool flush_now = group_start && q > 0, flush_first = flush_now && group_end;  // (as warp 0)
            if (flush_first) {
                flush(G - 1);
                __syncwarp();
                if (lane == 0) mbar_arrive(&acc_free[(G - 1) & 1]);
            }
            const int st = q % kRaw;
            mbar_wait(&mb_raw[st], (uint32_t)(q / kRaw) & 1u);
            if (q >= 2) mbar_wait(&mb_mma[q & 1], (uint32_t)((q >> 1) - 1) & 1u);
            char* a_hi = split0 + (size_t)(q & 1) * kSplitBuf;
            const int kvalid = min(kGemmKc, kend - (kbeg + q * kGemmKc));
            raw_split<kGemmM, kSplitThr>(true, raw_a(st), a_hi, a_hi + kABytes, kvalid, do_rsum ? rsf : nullptr, lda, t);
            raw_split<NT, kSplitThr>(true, raw_b(st), a_hi + 2 * kABytes, a_hi + 2 * kABytes + kBBytes, kvalid,
                                     nullptr, ldb, t);
            fence_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&split_full[q & 1]);
            if (do_rsum && group_end) {
#pragma unroll
                for (int i = 0; i < kRsIt; ++i) {
                    rsum[i] += (double)rsf[i];
                    rsf[i] = 0.f;
                }
            }
            if (flush_now && !flush_first) {
                flush(G - 1);
                __syncwarp();
                if (lane == 0) mbar_arrive(&acc_free[(G - 1) & 1]);
            }
        }
    }
    if (nck > 0) flush(G);  // the last group
    __syncthreads();
    // ---- epilogue: this slice's partial D (no bias / ReLU / gate in a weight gradient) ----
    float* C = g.C + (int64_t)slice * g.slice_stride;
    const int m = (warp & 3) * 32 + lane;
    if (epi_warp && m < g.M) {
        float* crow = C + (int64_t)m * g.ldc;
#pragma unroll
        for (int j = 0; j < kColHalf; ++j)
            if (col0 + j < g.N) crow[col0 + j] = acc[j];
    }
    if (do_rsum) {  // per row: the partials of the threads that split its k groups, in a fixed order
        double* red = reinterpret_cast<double*>(raw0);  // [k group][row] (the ring is idle now)
        constexpr int rq_n = kGemmM / 4;
        if (warp > 0) {
            const int t = tid - 32;
#pragma unroll
            for (int it = 0; it < kRsIt; ++it) {
                const int idx = t + it * kSplitThr;
                if (idx >= kGemmM * 8) break;
                const int kq = idx & 3, rq = (idx >> 2) % rq_n, kb = (idx >> 2) / rq_n;
                red[kb * kGemmM + 4 * rq + kq] = rsum[it];
            }
        }
        __syncthreads();
        if (tid < g.M) {
            double tsum = 0.0;
            for (int kb = 0; kb < kGemmKc / 4; ++kb) tsum += red[kb * kGemmM + tid];
            g.rowsum[(int64_t)slice * g.M + tid] = (float)tsum;
        }
    }
    tc_before_sync();
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols) : "memory");
}

// out[i] (+)= sum_s part[s * stride + i], in fp64 in a fixed order (deterministic).  A block
// takes 32 consecutive outputs (coalesced 128-byte rows of each slice) x 8 slice groups; the
// 8 group partials are added in group order.
__global__ void __launch_bounds__(256) k_reduce_slices(const float* __restrict__ part, int slices, int64_t stride,
                                                       int64_t n, float* __restrict__ out, int accumulate) {
    __shared__ double red[8][33];
    const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
    for (int64_t i0 = (int64_t)blockIdx.x * 32; i0 < n; i0 += (int64_t)gridDim.x * 32) {
        const int64_t i = i0 + lane;
        double s = 0.0;
        if (i < n)
            for (int k = grp; k < slices; k += 8) s += part[k * stride + i];
        red[grp][lane] = s;
        __syncthreads();
        if (grp == 0 && i < n) {
            double t = 0.0;
#pragma unroll
            for (int g = 0; g < 8; ++g) t += red[g][lane];
            out[i] = accumulate ? out[i] + (float)t : (float)t;
        }
        __syncthreads();
    }
}

template <int NT, bool F, bool R>
void gemm_attr() {
    cudaFuncSetAttribute(k_gemm_tf32x3<NT, F, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, kGemmMaxSmem);
}

template <bool F, bool R>
int gemm_dispatch(const GemmArgs& g, dim3 grid, const GemmPlan& p, cudaStream_t st) {
    const size_t bytes = p.bytes;
    if (g.N <= 16)
        k_gemm_tf32x3<16, F, R><<<grid, kGemmThreads, bytes, st>>>(g, p.raw);
    else if (g.N <= 32)
        k_gemm_tf32x3<32, F, R><<<grid, kGemmThreads, bytes, st>>>(g, p.raw);
    else if (g.N <= 64)
        k_gemm_tf32x3<64, F, R><<<grid, kGemmThreads, bytes, st>>>(g, p.raw);
    else if (g.N <= 128)
        k_gemm_tf32x3<128, F, R><<<grid, kGemmThreads, bytes, st>>>(g, p.raw);
    else
        return -1;
    return 1;
}

template <bool F, bool R>
void gemm_attrs() {
    gemm_attr<16, F, R>(); gemm_attr<32, F, R>(); gemm_attr<64, F, R>(); gemm_attr<128, F, R>();
}

int launch_gemm_tf32x3(const GemmArgs& g, int slices, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        gemm_attrs<false, false>(); gemm_attrs<false, true>(); gemm_attrs<true, false>(); gemm_attrs<true, true>();
        cudaFuncSetAttribute(k_gemm_ws<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, kGemmMaxSmem);
        cudaFuncSetAttribute(k_gemm_ws<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, kGemmMaxSmem);
        cudaFuncSetAttribute(k_gemm_ws<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, kGemmMaxSmem);
        cudaFuncSetAttribute(k_gemm_ws<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, kGemmMaxSmem);
        cudaFuncSetAttribute(k_gemm_wsf<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, kGemmMaxSmem);
        cudaFuncSetAttribute(k_gemm_wsf<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, kGemmMaxSmem);
        cudaFuncSetAttribute(k_gemm_wsf<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, kGemmMaxSmem);
        cudaFuncSetAttribute(k_gemm_wsf<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, kGemmMaxSmem);
        attr = true;
    }
    if (g.M <= 0 || g.N <= 0) return 0;
    const int ntiles = (g.M + kGemmM - 1) / kGemmM;
    const int nt = g.N <= 16 ? 16 : g.N <= 32 ? 32 : g.N <= 64 ? 64 : 128;
    const int kps = std::min(g.k_per_slice, std::max(g.K, 0));
    const int nck = (kps + kGemmKc - 1) / kGemmKc;
    const int gx = std::min(ntiles, std::max(1, 148 / std::max(1, slices)));
    const dim3 grid(gx, std::max(1, slices));
    const bool flush = g.k_per_slice > kFlushChunks * kGemmKc;
    GemmPlan p = gemm_plan(nt, nck, ntiles > gx, g.a_m == 1, g.b_n == 1, flush);
    static const int raw_cap = [] {  // TSB_GEMM_RAW: cap on the raw stages (A/B timing)
        const char* e = std::getenv("TSB_GEMM_RAW");
        return e ? std::atoi(e) : kMaxRaw;
    }();
    if (p.raw > raw_cap && raw_cap >= 2) {
        p.raw = raw_cap;
        p.bytes = gemm_bytes(nt, nck, p.b_res, g.a_m == 1, g.b_n == 1, p.raw, flush && !p.b_res ? 2 : 1);
    }
    static const bool ws_off = [] {  // TSB_GEMM_WS=0: the single-role kernel (A/B timing)
        const char* e = std::getenv("TSB_GEMM_WS");
        return e && e[0] == '0';
    }();
    const bool ws = !flush && p.b_res && nck > 0 && slices <= 1 && g.K <= g.k_per_slice && !ws_off;
    if (g.chain_x && (!ws || nt != 128 || g.N < 63)) return kGemmNoChain;
    if (ws) {
        GemmPlan pw = p;  // the epilogue's staging blocks come after the raw ring
        while (pw.raw > 2 && pw.bytes + kEpiStageBytes > (size_t)kGemmMaxSmem) {
            --pw.raw;
            pw.bytes = gemm_bytes(nt, nck, true, g.a_m == 1, g.b_n == 1, pw.raw);
        }
        const size_t bytes = pw.bytes + kEpiStageBytes;
        p = pw;
        if (nt == 16) k_gemm_ws<16><<<grid, kGemmThreads, bytes, st>>>(g, p.raw);
        else if (nt == 32) k_gemm_ws<32><<<grid, kGemmThreads, bytes, st>>>(g, p.raw);
        else if (nt == 64) k_gemm_ws<64><<<grid, kGemmThreads, bytes, st>>>(g, p.raw);
        else k_gemm_ws<128><<<grid, kGemmThreads, bytes, st>>>(g, p.raw);
        return 1;
    }
    static const bool wsf_off = [] {  // TSB_GEMM_WSF=0: the single-role kernel (A/B timing)
        const char* e = std::getenv("TSB_GEMM_WSF");
        return e && e[0] == '0';
    }();
    const bool bulk_ok = g.a_m == 1 && g.b_n == 1 && g.M <= g.a_k && g.a_k <= kGemmM && g.N <= g.b_k && g.b_k <= nt &&
                         ((g.a_k | g.b_k) & 3) == 0 && (((uintptr_t)g.A | (uintptr_t)g.B) & 15) == 0;
    if (flush && !p.b_res && bulk_ok && g.M <= kGemmM && !wsf_off) {
        const size_t bytes = p.bytes;
        if (nt == 16) k_gemm_wsf<16><<<grid, kGemmThreads, bytes, st>>>(g, p.raw);
        else if (nt == 32) k_gemm_wsf<32><<<grid, kGemmThreads, bytes, st>>>(g, p.raw);
        else if (nt == 64) k_gemm_wsf<64><<<grid, kGemmThreads, bytes, st>>>(g, p.raw);
        else k_gemm_wsf<128><<<grid, kGemmThreads, bytes, st>>>(g, p.raw);
        return 1;
    }
    if (flush) return p.b_res ? gemm_dispatch<true, true>(g, grid, p, st) : gemm_dispatch<true, false>(g, grid, p, st);
    return p.b_res ? gemm_dispatch<false, true>(g, grid, p, st) : gemm_dispatch<false, false>(g, grid, p, st);
}

void launch_reduce_slices(const float* part, int slices, int64_t stride, int64_t n, float* out, bool accumulate,
                          cudaStream_t st) {
    if (n <= 0) return;
    const int grid = (int)std::min<int64_t>((n + 31) / 32, 148 * 8);
    k_reduce_slices<<<grid, 256, 0, st>>>(part, slices, stride, n, out, accumulate ? 1 : 0);
}

}  // namespace tsb

namespace tsb {

// ---------------------------------------------------------------------------
// DeformNet helpers (deform.cpp:10-26, 60-78, 142-155)
// ---------------------------------------------------------------------------

// X[n][c * ex + j] = gamma_j(pos_c / coord_scale), then the (shared) time encoding.
// gamma = [v, sin(pi 2^l v), cos(pi 2^l v)] in fp64, rounded once.
__global__ void k_deform_encode(const float* __restrict__ pos, int64_t pos_stride, int64_t n, double inv_scale,
                                int l_x, DeformEnc te, float* __restrict__ X, int64_t ldx) {
    const int ex = 1 + 2 * l_x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        float* row = X + i * ldx;
        for (int c = 0; c < 3; ++c) {
            const double v = (double)pos[i * pos_stride + c] * inv_scale;
            float* o = row + c * ex;
            o[0] = (float)v;
            double s, co;
            sincospi(v, &s, &co);
            for (int l = 0; l < l_x; ++l) {
                if (l) sincospi_double(s, co);
                o[1 + 2 * l] = (float)s;
                o[2 + 2 * l] = (float)co;
            }
        }
        for (int j = 0; j < te.n; ++j) row[3 * ex + j] = te.v[j];
    }
}

// d_pos[i][c] += sum_j gamma'_j(v_c) d_input[i][c * ex + j] / coord_scale (v_c = X[i][c * ex]).
__global__ void k_deform_chain(const float* __restrict__ d_input, int64_t ldd, const float* __restrict__ X,
                               int64_t ldx, int64_t n, double inv_scale, int l_x, float* __restrict__ d_pos,
                               int64_t dpos_stride, int accumulate) {
    const int ex = 1 + 2 * l_x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        for (int c = 0; c < 3; ++c) {
            const float* din = d_input + i * ldd + c * ex;
            const double v = (double)X[i * ldx + c * ex];
            double acc = din[0];
            double fr = M_PI, s, co;
            sincospi(v, &s, &co);
            for (int l = 0; l < l_x; ++l, fr *= 2.0) {
                if (l) sincospi_double(s, co);
                acc += fr * co * (double)din[1 + 2 * l] - fr * s * (double)din[2 + 2 * l];
            }
            float* o = d_pos + i * dpos_stride + c;
            const float val = (float)(acc * inv_scale);
            *o = accumulate ? *o + val : val;
        }
    }
}

void launch_deform_encode(const float* pos, int64_t pos_stride, int64_t n, double inv_scale, int l_x,
                          const DeformEnc& te, float* X, int64_t ldx, cudaStream_t st) {
    if (n <= 0) return;
    const int grid = (int)std::min<int64_t>((n + 127) / 128, 148 * 16);
    k_deform_encode<<<grid, 128, 0, st>>>(pos, pos_stride, n, inv_scale, l_x, te, X, ldx);
}

void launch_deform_chain(const float* d_input, int64_t ldd, const float* X, int64_t ldx, int64_t n, double inv_scale,
                         int l_x, float* d_pos, int64_t dpos_stride, bool accumulate, cudaStream_t st) {
    if (n <= 0) return;
    const int grid = (int)std::min<int64_t>((n + 127) / 128, 148 * 16);
    k_deform_chain<<<grid, 128, 0, st>>>(d_input, ldd, X, ldx, n, inv_scale, l_x, d_pos, dpos_stride,
                                         accumulate ? 1 : 0);
}

}  // namespace tsb

// ===========================================================================
// Fused DeformNet forward: one persistent CTA per SM walks 128-row tiles; the
// tile's activations never leave the SM.  Per tile: positional encoding -> A
// (3xTF32 hi/lo, canonical K-major, shared memory) -> for every layer the
// tensor core accumulates A x W_l^T in TMEM while the weights stream through a
// 3-stage shared-memory ring by bulk copies (cp.async.bulk + mbarrier
// complete_tx) from a pre-split, pre-laid-out copy (k_pack_weights); the
// epilogue adds the bias, applies ReLU, optionally stores the activation for the
// backward, and writes it back split into A for the next layer.  The last
// layer's 3 outputs go to `out`.
// ===========================================================================
namespace tsb {
namespace {
constexpr int kMlpThreads = 512;  // 16 warps: the epilogue is latency-bound
constexpr int kMlpStages = 3;
constexpr uint32_t kMlpASbo = (128 / 4) * kCoreBytes;          // A tile: K extent 128 -> 4096 B per 8-row group
constexpr uint32_t kMlpAHalf = 128 * 128 * 4;                  // hi (then lo) A buffer
constexpr uint32_t kMlpStageBytes = 128 * kGemmKc * 4 * 2;     // largest weight chunk (N = 128, hi + lo)

__device__ __forceinline__ uint32_t a_off(int r, int k) {
    return (uint32_t)(r >> 3) * kMlpASbo + (uint32_t)(k >> 2) * kCoreBytes + (uint32_t)(r & 7) * 16u +
           (uint32_t)(k & 3) * 4u;
}

// 3xTF32 split for operands held in shared memory: hi = tf32(x) (round to nearest), lo =
// x - hi exactly (the tensor core truncates lo to tf32, an error below 2^-21 |x|), so hi +
// lo reproduces x and the activations can be stored from the A buffer without a copy.
__device__ __forceinline__ void split_exact(float x, float& hi, float& lo) {
    uint32_t h;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
    hi = __uint_as_float(h);
    lo = x - hi;
}
__device__ __forceinline__ void split_exact(double x, float& hi, float& lo) { split_exact((float)x, hi, lo); }

// rows m0 .. m0+127 (< n), columns [0, ncols) of the A tile -> dst[m * ld + c], coalesced:
// per iteration a warp covers 8 rows x 4 consecutive column quads (no index division).
// Warps w0 .. w0 + nwarps - 1 take part (the MMA-issuing warp 0 does not while it issues).
__device__ __forceinline__ void store_rows(const char* A_hi, const char* A_lo, float* dst, int64_t ld, int64_t m0,
                                           int64_t n, int ncols, uint32_t* bits, int w0, int nwarps) {
    const int lane = threadIdx.x & 31, warp = (int)(threadIdx.x >> 5) - w0;
    const int r8 = lane & 7, qi = lane >> 3, nq = ncols / 4;
    // bits (ncols a multiple of 32): the ReLU gates, word w of a row = columns 32 w .. 32 w + 31;
    // the 4 lanes of a row hold 16 consecutive columns per step
    const int64_t ldw = ncols / 32;
    for (int rg = warp; rg < 16; rg += nwarps) {
        const int r = rg * 8 + r8;
        const int64_t m = m0 + r;
        const bool rv = m < n;
        float* row = dst + m * ld;
        const bool al = (((uintptr_t)row) & 15) == 0;
        uint32_t word = 0;
        for (int q = qi, t = 0; q < nq; q += 4, ++t) {
            const float4 h = *reinterpret_cast<const float4*>(A_hi + a_off(r, 4 * q));
            const float4 l = *reinterpret_cast<const float4*>(A_lo + a_off(r, 4 * q));
            const float4 v = make_float4(h.x + l.x, h.y + l.y, h.z + l.z, h.w + l.w);
            if (rv) {
                if (al) {
                    *reinterpret_cast<float4*>(row + 4 * q) = v;
                } else {
                    row[4 * q] = v.x; row[4 * q + 1] = v.y; row[4 * q + 2] = v.z; row[4 * q + 3] = v.w;
                }
            }
            if (bits) {  // (warp-uniform: every lane of the warp runs nq / 4 steps)
                uint32_t nib = (v.x > 0.f ? 1u : 0u) | (v.y > 0.f ? 2u : 0u) | (v.z > 0.f ? 4u : 0u) |
                               (v.w > 0.f ? 8u : 0u);
                nib <<= 4 * qi;
                nib |= __shfl_xor_sync(0xffffffffu, nib, 8);
                nib |= __shfl_xor_sync(0xffffffffu, nib, 16);
                word |= nib << (16 * (t & 1));
                if (t & 1) {
                    if (qi == 0 && rv) bits[m * ldw + (t >> 1)] = word;
                    word = 0;
                }
            }
        }
        if (qi == 0 && rv)
            for (int c = 4 * nq; c < ncols; ++c)
                row[c] = *reinterpret_cast<const float*>(A_hi + a_off(r, c)) +
                         *reinterpret_cast<const float*>(A_lo + a_off(r, c));
    }
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* mbar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(mbar))
        : "memory");
}
}  // namespace

// W_l (rows x cols, row-major, inside the flat parameters) -> per 32-wide K chunk a
// block [hi | lo] of NT_l x 32 tf32 in the canonical K-major layout (zero padded).
__global__ void k_pack_weights(MlpLayout lay, const float* __restrict__ params, char* __restrict__ out) {
    const int l = blockIdx.y;
    if (l >= lay.layers) return;
    const int nt = lay.nt[l], rows = lay.rows[l], cols = lay.cols[l];
    const int nchunks = lay.chunks[l];
    const float* W = params + lay.w_off[l];
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < nchunks * nt * kGemmKc;
         idx += gridDim.x * blockDim.x) {
        const int c = idx / (nt * kGemmKc), rem = idx - c * nt * kGemmKc;
        const int n = rem / kGemmKc, k = rem - n * kGemmKc, gk = c * kGemmKc + k;
        const float w = (n < rows && gk < cols) ? W[(int64_t)n * cols + gk] : 0.f;
        float h, lo;
        split_tf32(w, h, lo);
        char* blk = out + lay.chunk_off[l] + (int64_t)c * nt * kGemmKc * 8;
        const uint32_t o = core_off(n, k);
        *reinterpret_cast<float*>(blk + o) = h;
        *reinterpret_cast<float*>(blk + (int64_t)nt * kGemmKc * 4 + o) = lo;
    }
}

__device__ __forceinline__ void bar_compute() { asm volatile("bar.sync 1, %0;" ::"n"(kMlpThreads) : "memory"); }

// kMlpThreads compute threads (thread 0 issues the MMAs) + one producer warp whose lane 0
// streams the weight chunks into the ring as stages free up (the MMA issuer never waits
// for the tensor core, only for data).
__global__ void __launch_bounds__(kMlpThreads + 32, 1) k_mlp_fwd_fused(MlpFwdArgs a) {
    extern __shared__ __align__(1024) char smem[];
    __shared__ __align__(8) uint64_t mb_full[kMlpStages], mb_empty[kMlpStages], mb_layer;
    __shared__ uint32_t tmem_base_s;
    char* A_hi = smem;
    char* A_lo = smem + kMlpAHalf;
    char* ring = smem + 2 * kMlpAHalf;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const MlpLayout& lay = a.lay;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tmem_base_s))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        for (int i = 0; i < kMlpStages; ++i) {
            mbar_init(&mb_full[i], 1);
            mbar_init(&mb_empty[i], 1);
        }
        mbar_init(&mb_layer, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    const uint32_t tmem = tmem_base_s;
    const uint32_t tl = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    const int ntiles = (int)((a.n + 127) / 128);
    const int my_tiles = ntiles > (int)blockIdx.x ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    const uint32_t total = (uint32_t)my_tiles * (uint32_t)lay.total_chunks;  // weight chunks this CTA consumes

    // chunk q of this CTA -> (layer, chunk in layer)
    auto chunk_src = [&](uint32_t q, uint32_t& bytes) -> const char* {
        const uint32_t local = q % (uint32_t)lay.total_chunks;
        int l = 0;
        uint32_t base = 0;
        while (local >= base + (uint32_t)lay.chunks[l]) {
            base += lay.chunks[l];
            ++l;
        }
        bytes = (uint32_t)lay.nt[l] * kGemmKc * 8u;
        return a.wpack + lay.chunk_off[l] + (int64_t)(local - base) * bytes;
    };
    if (warp == kMlpThreads / 32) {  // ---- producer warp ----
        if (lane == 0)
            for (uint32_t q = 0; q < total; ++q) {
                const int st = (int)(q % kMlpStages);
                if (q >= (uint32_t)kMlpStages) mbar_wait(&mb_empty[st], ((q / kMlpStages) - 1) & 1u);
                uint32_t bytes;
                const char* src = chunk_src(q, bytes);
                bulk_g2s(ring + (size_t)st * kMlpStageBytes, src, bytes, &mb_full[st]);
            }
        __syncwarp();
    } else {

    uint32_t q = 0;          // next chunk to consume
    uint32_t lphase = 0;     // mb_layer completions
    const int ex = 1 + 2 * a.l_x;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t m0 = (int64_t)tile * 128;
        // ---- positional encoding of the tile's rows (four threads per row: x, y, z, time + padding) ----
        {
            const int r = tid & 127, part = tid >> 7;
            const int64_t m = m0 + r;
            const int kb = part * ex;
            if (part < 3) {
                const double v = m < a.n ? (double)a.pos[m * a.pos_stride + part] * a.inv_scale : 0.0;
                float h, lo;
                split_exact(v, h, lo);
                *reinterpret_cast<float*>(A_hi + a_off(r, kb)) = h;
                *reinterpret_cast<float*>(A_lo + a_off(r, kb)) = lo;
                double sn, co;
                sincospi(v, &sn, &co);
                for (int l = 0; l < a.l_x; ++l) {
                    if (l) sincospi_double(sn, co);
                    split_exact(sn, h, lo);
                    *reinterpret_cast<float*>(A_hi + a_off(r, kb + 1 + 2 * l)) = h;
                    *reinterpret_cast<float*>(A_lo + a_off(r, kb + 1 + 2 * l)) = lo;
                    split_exact(co, h, lo);
                    *reinterpret_cast<float*>(A_hi + a_off(r, kb + 2 + 2 * l)) = h;
                    *reinterpret_cast<float*>(A_lo + a_off(r, kb + 2 + 2 * l)) = lo;
                }
            } else {
                for (int k = kb; k < lay.cols_pad[0]; ++k) {
                    const float x = k - kb < a.te.n ? a.te.v[k - kb] : 0.f;
                    float h, lo;
                    split_exact(x, h, lo);
                    *reinterpret_cast<float*>(A_hi + a_off(r, k)) = h;
                    *reinterpret_cast<float*>(A_lo + a_off(r, k)) = lo;
                }
            }
        }
        fence_async_smem();
        bar_compute();

        for (int l = 0; l < lay.layers; ++l) {
            const int nt = lay.nt[l];
            // A holds this layer's input (read-only until its epilogue): warps 1-15 store it for
            // the backward -- the encoding (X) or the previous layer's activation (H, + its ReLU
            // gates as bits: the backward's gate reads 1 bit instead of the activation) -- while
            // thread 0 issues the layer's MMAs
            const bool store_x = l == 0 && a.X;
            const bool store_h = l > 0 && a.H[l - 1];
            if (warp > 0) {
                if (store_x) store_rows(A_hi, A_lo, a.X, a.ldx, m0, a.n, a.din, nullptr, 1, kMlpThreads / 32 - 1);
                if (store_h)
                    store_rows(A_hi, A_lo, a.H[l - 1], a.ldh, m0, a.n, lay.nt[l - 1], a.Hbits[l - 1], 1,
                               kMlpThreads / 32 - 1);
            }
            if (tid == 0) {
                tc_after_sync();
                const uint32_t idesc = idesc_tf32(128, nt);
                const uint32_t ah = smem_u32(A_hi), al = smem_u32(A_lo);
                for (int c = 0; c < lay.chunks[l]; ++c, ++q) {
                    const int st = (int)(q % kMlpStages);
                    mbar_wait(&mb_full[st], (q / kMlpStages) & 1u);
                    const uint32_t bh = smem_u32(ring + (size_t)st * kMlpStageBytes);
                    const uint32_t bl = bh + (uint32_t)nt * kGemmKc * 4;
#pragma unroll
                    for (int s = 0; s < kGemmKc / 8; ++s) {
                        const uint32_t aoff = (uint32_t)(c * (kGemmKc / 4) + 2 * s) * kCoreBytes;
                        const uint32_t boff = (uint32_t)(2 * s) * kCoreBytes;
                        const uint64_t dah = umma_desc(ah + aoff, kCoreBytes, kMlpASbo);
                        const uint64_t dal = umma_desc(al + aoff, kCoreBytes, kMlpASbo);
                        const uint64_t dbh = umma_desc(bh + boff, kCoreBytes, kGroupBytes);
                        const uint64_t dbl = umma_desc(bl + boff, kCoreBytes, kGroupBytes);
                        mma_tf32(tmem, dah, dbh, idesc, (c > 0 || s > 0) ? 1u : 0u);
                        mma_tf32(tmem, dah, dbl, idesc, 1u);
                        mma_tf32(tmem, dal, dbh, idesc, 1u);
                    }
                    mma_commit(&mb_empty[st]);
                }
                mma_commit(&mb_layer);
            } else if (tid != 0) {
                q += lay.chunks[l];
            }
            mbar_wait(&mb_layer, lphase & 1u);
            ++lphase;
            if (store_x || store_h) bar_compute();  // the epilogue overwrites A
            tc_after_sync();
            // ---- epilogue: bias, ReLU; split back into A for the next layer ----
            const int r = (warp & 3) * 32 + lane;
            const int64_t m = m0 + r;
            const float* bias = a.params + lay.b_off[l];
            const bool hidden = l + 1 < lay.layers;
            if (hidden) {
                const int q4 = nt / 4, c0 = (warp >> 2) * q4;
                for (int cc = 0; cc < q4; cc += 16) {
                    uint32_t v[16];
                    tmem_ld16(tl + (uint32_t)(c0 + cc), v);
#pragma unroll
                    for (int j = 0; j < 16; j += 4) {
                        const int col = c0 + cc + j;
                        float4 x;
                        x.x = fmaxf(__uint_as_float(v[j]) + __ldg(bias + col), 0.f);
                        x.y = fmaxf(__uint_as_float(v[j + 1]) + __ldg(bias + col + 1), 0.f);
                        x.z = fmaxf(__uint_as_float(v[j + 2]) + __ldg(bias + col + 2), 0.f);
                        x.w = fmaxf(__uint_as_float(v[j + 3]) + __ldg(bias + col + 3), 0.f);
                        float4 h, lo;
                        split_exact(x.x, h.x, lo.x);
                        split_exact(x.y, h.y, lo.y);
                        split_exact(x.z, h.z, lo.z);
                        split_exact(x.w, h.w, lo.w);
                        *reinterpret_cast<float4*>(A_hi + a_off(r, col)) = h;
                        *reinterpret_cast<float4*>(A_lo + a_off(r, col)) = lo;
                    }
                }
            } else if (warp < 4) {
                uint32_t v[16];
                tmem_ld16(tl, v);
                if (m < a.n)
                    for (int j = 0; j < 3; ++j) a.out[m * a.out_stride + j] = __uint_as_float(v[j]) + __ldg(bias + j);
            }
            fence_async_smem();
            tc_before_sync();
            bar_compute();
        }
    }
    }  // compute threads
    tc_before_sync();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem) : "memory");
}

// ---------------------------------------------------------------------------
// The same forward with the activations in tensor memory.  The layer input A (hi / lo) is
// the MMA's A operand read from TMEM (tcgen05.mma ... [a-tmem]): the epilogue moves the
// accumulator D -> registers (bias, ReLU, split) -> A with tcgen05.st, so shared memory
// holds only the weight ring, which is then deep enough (7 stages of 32 K-columns) to keep
// the tensor core fed from L2.  TMEM: D at column 0, A hi at 128, A lo at 256 (512
// allocated, one CTA per SM).  The activations the backward reads (encoding X, hidden H
// + ReLU gate bits) go to global memory straight from the epilogue's registers.
// ---------------------------------------------------------------------------
constexpr int kMlpStagesT = 4;
constexpr int kStgLd = 132;  // fp32 staging tile row stride (floats): the layer input, stored for the backward
constexpr uint32_t kTmA = 128, kTmAlo = 256;  // TMEM column offsets

__device__ __forceinline__ void mma_tf32_at(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                            uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}
__device__ __forceinline__ void tmem_st1(uint32_t taddr, uint32_t v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(v) : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }


// Rows m0 .. m0+127 (< n), columns [0, ncols) of the fp32 staging tile -> dst[m * ld + c], one
// row per warp instruction (coalesced), + the ReLU gate bits (ncols a multiple of 32).
__device__ __forceinline__ void store_staged(const float* S, float* dst, int64_t ld, int64_t m0, int64_t n, int ncols,
                                             uint32_t* bits, int w0, int nwarps) {
    const int lane = threadIdx.x & 31, warp = (int)(threadIdx.x >> 5) - w0;
    const int nq = ncols / 4;
    const int64_t ldw = ncols / 32;
    for (int rr = warp; rr < 128; rr += nwarps) {
        const int64_t m = m0 + rr;
        if (m >= n) break;
        const float* srow = S + rr * kStgLd;
        float* drow = dst + m * ld;
        const bool al = ((((uintptr_t)drow) | (ld * 4)) & 15) == 0;
        for (int q0 = 0; q0 < nq; q0 += 32) {
            const int q = q0 + lane;
            const float4 v = q < nq ? *reinterpret_cast<const float4*>(srow + 4 * q) : make_float4(0.f, 0.f, 0.f, 0.f);
            if (q < nq) {
                if (al) {
                    *reinterpret_cast<float4*>(drow + 4 * q) = v;
                } else {
                    drow[4 * q] = v.x; drow[4 * q + 1] = v.y; drow[4 * q + 2] = v.z; drow[4 * q + 3] = v.w;
                }
            }
            if (bits) {
                uint32_t nib = (v.x > 0.f ? 1u : 0u) | (v.y > 0.f ? 2u : 0u) | (v.z > 0.f ? 4u : 0u) | (v.w > 0.f ? 8u : 0u);
                nib <<= 4 * (lane & 7);
                nib |= __shfl_xor_sync(0xffffffffu, nib, 1);
                nib |= __shfl_xor_sync(0xffffffffu, nib, 2);
                nib |= __shfl_xor_sync(0xffffffffu, nib, 4);
                if ((lane & 7) == 0 && q < nq) bits[m * ldw + q / 8] = nib;
            }
        }
    }
}

// kMlpThreads compute threads (thread 0 issues the MMAs) + one producer warp whose lane 0
// streams the weight chunks into the ring as stages free up (the MMA issuer never waits
// for the tensor core, only for data).
__global__ void __launch_bounds__(kMlpThreads + 32, 1) k_mlp_fwd_tm(MlpFwdArgs a) {
    extern __shared__ __align__(1024) char smem[];
    __shared__ __align__(8) uint64_t mb_full[kMlpStagesT], mb_empty[kMlpStagesT], mb_layer;
    __shared__ uint32_t tmem_base_s;
    char* ring = smem;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const MlpLayout& lay = a.lay;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base_s))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        for (int i = 0; i < kMlpStagesT; ++i) {
            mbar_init(&mb_full[i], 1);
            mbar_init(&mb_empty[i], 1);
        }
        mbar_init(&mb_layer, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    const uint32_t tmem = tmem_base_s;
    const uint32_t tl = tmem + ((uint32_t)((warp & 3) * 32) << 16);  // this warp's lane quadrant
    const int wg = warp >> 2;                                          // column group (0..3)
    const int ntiles = (int)((a.n + 127) / 128);
    const int my_tiles = ntiles > (int)blockIdx.x ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    const uint32_t total = (uint32_t)my_tiles * (uint32_t)lay.total_chunks;

    auto chunk_src = [&](uint32_t q, uint32_t& bytes) -> const char* {
        const uint32_t local = q % (uint32_t)lay.total_chunks;
        int l = 0;
        uint32_t base = 0;
        while (local >= base + (uint32_t)lay.chunks[l]) {
            base += lay.chunks[l];
            ++l;
        }
        bytes = (uint32_t)lay.nt[l] * kGemmKc * 8u;
        return a.wpack + lay.chunk_off[l] + (int64_t)(local - base) * bytes;
    };
    if (warp == kMlpThreads / 32) {  // ---- producer warp ----
        if (lane == 0)
            for (uint32_t q = 0; q < total; ++q) {
                const int st = (int)(q % kMlpStagesT);
                if (q >= (uint32_t)kMlpStagesT) mbar_wait(&mb_empty[st], ((q / kMlpStagesT) - 1) & 1u);
                uint32_t bytes;
                const char* src = chunk_src(q, bytes);
                bulk_g2s(ring + (size_t)st * kMlpStageBytes, src, bytes, &mb_full[st]);
            }
        __syncwarp();
    } else {

    uint32_t q = 0, lphase = 0;
    const int ex = 1 + 2 * a.l_x;
    const int kpad0 = lay.chunks[0] * kGemmKc;
    float* S = reinterpret_cast<float*>(smem + (size_t)kMlpStagesT * kMlpStageBytes);  // [128][kStgLd]
    const int r = (warp & 3) * 32 + lane;  // = the TMEM lane this thread may access
    float* srow = S + r * kStgLd;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t m0 = (int64_t)tile * 128;
        const int64_t m = m0 + r;
        const bool rv = m < a.n;
        // ---- positional encoding of the tile's rows into the staging tile (warp group: x, y, z,
        //      time + zero padding), then A = split(staging) into TMEM ----
        {
            const int kb = wg * ex;
            if (wg < 3) {
                const double v = rv ? (double)a.pos[m * a.pos_stride + wg] * a.inv_scale : 0.0;
                srow[kb] = (float)v;
                double sn, co;
                sincospi(v, &sn, &co);
                for (int l = 0; l < a.l_x; ++l) {
                    if (l) sincospi_double(sn, co);
                    srow[kb + 1 + 2 * l] = (float)sn;
                    srow[kb + 2 + 2 * l] = (float)co;
                }
            } else {
                for (int k = kb; k < kpad0; ++k) srow[k] = k - kb < a.te.n ? a.te.v[k - kb] : 0.f;
            }
            bar_compute();
            for (int ch = wg; ch < kpad0 / 16; ch += 4) {
                uint32_t hv[16], lv[16];
#pragma unroll
                for (int j = 0; j < 16; j += 4) {
                    const float4 x = *reinterpret_cast<const float4*>(srow + ch * 16 + j);
                    float h, lo;
                    split_exact(x.x, h, lo); hv[j] = __float_as_uint(h); lv[j] = __float_as_uint(lo);
                    split_exact(x.y, h, lo); hv[j + 1] = __float_as_uint(h); lv[j + 1] = __float_as_uint(lo);
                    split_exact(x.z, h, lo); hv[j + 2] = __float_as_uint(h); lv[j + 2] = __float_as_uint(lo);
                    split_exact(x.w, h, lo); hv[j + 3] = __float_as_uint(h); lv[j + 3] = __float_as_uint(lo);
                }
                tmem_st16(tl + kTmA + (uint32_t)(ch * 16), hv);
                tmem_st16(tl + kTmAlo + (uint32_t)(ch * 16), lv);
            }
            tmem_st_wait();
        }
        tc_before_sync();
        bar_compute();

        for (int l = 0; l < lay.layers; ++l) {
            const int nt = lay.nt[l];
            // the staging tile holds this layer's input: warps 1-15 store it for the backward
            // (X, or H of the layer below + its ReLU gate bits) while thread 0 issues the MMAs
            if (warp > 0) {
                if (l == 0 && a.X) store_staged(S, a.X, a.ldx, m0, a.n, a.din, nullptr, 1, kMlpThreads / 32 - 1);
                if (l > 0 && a.H[l - 1])
                    store_staged(S, a.H[l - 1], a.ldh, m0, a.n, lay.rows[l - 1], a.Hbits[l - 1], 1,
                                 kMlpThreads / 32 - 1);
            }
            if (tid == 0) {
                tc_after_sync();
                const uint32_t idesc = idesc_tf32(128, nt);
                for (int c = 0; c < lay.chunks[l]; ++c, ++q) {
                    const int st = (int)(q % kMlpStagesT);
                    mbar_wait(&mb_full[st], (q / kMlpStagesT) & 1u);
                    const uint32_t bh = smem_u32(ring + (size_t)st * kMlpStageBytes);
                    const uint32_t bl = bh + (uint32_t)nt * kGemmKc * 4;
#pragma unroll
                    for (int s = 0; s < kGemmKc / 8; ++s) {
                        const uint32_t k0 = (uint32_t)(c * kGemmKc + 8 * s);
                        const uint32_t boff = (uint32_t)(2 * s) * kCoreBytes;
                        const uint64_t dbh = umma_desc(bh + boff, kCoreBytes, kGroupBytes);
                        const uint64_t dbl = umma_desc(bl + boff, kCoreBytes, kGroupBytes);
                        mma_tf32_at(tmem, tmem + kTmA + k0, dbh, idesc, (c > 0 || s > 0) ? 1u : 0u);
                        mma_tf32_at(tmem, tmem + kTmA + k0, dbl, idesc, 1u);
                        mma_tf32_at(tmem, tmem + kTmAlo + k0, dbh, idesc, 1u);
                    }
                    mma_commit(&mb_empty[st]);
                }
                mma_commit(&mb_layer);
            } else {
                q += lay.chunks[l];
            }
            mbar_wait(&mb_layer, lphase & 1u);
            ++lphase;
            bar_compute();  // the staging tile is free again
            tc_after_sync();
            const float* bias = a.params + lay.b_off[l];
            const int rows = lay.rows[l];
            if (l + 1 < lay.layers) {
                // ---- hidden epilogue: D -> bias, ReLU -> staging (fp32) and A (split) for layer l + 1 ----
                const int kpn = lay.chunks[l + 1] * kGemmKc;  // the next layer's (padded) K
                for (int ch = wg; ch < kpn / 16; ch += 4) {
                    const int col = ch * 16;
                    uint32_t v[16], hv[16], lv[16];
                    float x[16];
                    if (col < nt) {
                        tmem_ld16(tl + (uint32_t)col, v);
#pragma unroll
                        for (int j = 0; j < 16; ++j)
                            x[j] = col + j < rows ? fmaxf(__uint_as_float(v[j]) + __ldg(bias + col + j), 0.f) : 0.f;
                    } else {
#pragma unroll
                        for (int j = 0; j < 16; ++j) x[j] = 0.f;
                    }
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        float h, lo;
                        split_exact(x[j], h, lo);
                        hv[j] = __float_as_uint(h);
                        lv[j] = __float_as_uint(lo);
                    }
#pragma unroll
                    for (int j = 0; j < 16; j += 4)
                        *reinterpret_cast<float4*>(srow + col + j) = make_float4(x[j], x[j + 1], x[j + 2], x[j + 3]);
                    tmem_st16(tl + kTmA + (uint32_t)col, hv);
                    tmem_st16(tl + kTmAlo + (uint32_t)col, lv);
                }
                tmem_st_wait();
            } else if (warp < 4) {
                uint32_t v[16];
                tmem_ld16(tl, v);
                if (rv)
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (j < rows) a.out[m * a.out_stride + j] = __uint_as_float(v[j]) + __ldg(bias + j);
            }
            tc_before_sync();
            bar_compute();
        }
    }
    }  // compute threads
    tc_before_sync();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

// ---------------------------------------------------------------------------
// Pipelined variant: layer l + 1's MMAs start on each 32-column K chunk of its input as soon
// as the epilogue of layer l has written it (instead of after the whole epilogue).  Layers
// alternate between two accumulators (TMEM: D0 0-127, D1 128-255, A hi 256-383, A lo
// 384-511), so layer l + 1 accumulates while layer l's is still being read.  Roles: warps
// 0-15 encode / epilogue / store the staging tile; warp 16 lane 0 streams the weights;
// warp 17 lane 0 issues the MMAs.
//   a_ready[c]  the 16 compute warps wrote A columns [32c, 32c + 32) of the next layer's
//               input (one barrier per chunk index: each completes once per layer, so a
//               parity wait cannot be lapped)
//   mb_layer    a layer's MMAs are done (its accumulator may be read)
// ---------------------------------------------------------------------------
constexpr uint32_t kTpD1 = 128, kTpA = 256, kTpAlo = 384;
constexpr int kMlpThreadsP = kMlpThreads + 64;

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t* v) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}

__global__ void __launch_bounds__(kMlpThreadsP, 1) k_mlp_fwd_tp(MlpFwdArgs a) {
    extern __shared__ __align__(1024) char smem[];
    __shared__ __align__(8) uint64_t mb_full[kMlpStagesT], mb_empty[kMlpStagesT], mb_layer, a_ready[4];
    __shared__ uint32_t tmem_base_s;
    char* ring = smem;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const MlpLayout& lay = a.lay;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base_s))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        for (int i = 0; i < kMlpStagesT; ++i) {
            mbar_init(&mb_full[i], 1);
            mbar_init(&mb_empty[i], 1);
        }
        mbar_init(&mb_layer, 1);
        for (int c = 0; c < 4; ++c) mbar_init(&a_ready[c], kMlpThreads / 32);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    const uint32_t tmem = tmem_base_s;
    const uint32_t tl = tmem + ((uint32_t)((warp & 3) * 32) << 16);  // this warp's lane quadrant
    const int wg = warp >> 2;                                          // column group (0..3)
    const int ntiles = (int)((a.n + 127) / 128);
    const int my_tiles = ntiles > (int)blockIdx.x ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    const uint32_t total = (uint32_t)my_tiles * (uint32_t)lay.total_chunks;

    if (warp == kMlpThreads / 32) {  // ---- weight producer ----
        if (lane == 0)
            for (uint32_t q = 0; q < total; ++q) {
                const int st = (int)(q % kMlpStagesT);
                if (q >= (uint32_t)kMlpStagesT) mbar_wait(&mb_empty[st], ((q / kMlpStagesT) - 1) & 1u);
                const uint32_t local = q % (uint32_t)lay.total_chunks;
                int l = 0;
                uint32_t base = 0;
                while (local >= base + (uint32_t)lay.chunks[l]) {
                    base += lay.chunks[l];
                    ++l;
                }
                const uint32_t bytes = (uint32_t)lay.nt[l] * kGemmKc * 8u;
                bulk_g2s(ring + (size_t)st * kMlpStageBytes, a.wpack + lay.chunk_off[l] + (int64_t)(local - base) * bytes,
                         bytes, &mb_full[st]);
            }
        __syncwarp();
    } else if (warp == kMlpThreads / 32 + 1) {  // ---- MMA issuer ----
        if (lane == 0) {
            uint32_t q = 0, aph = 0;  // aph: bit c = parity of a_ready[c]'s next completion
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                for (int l = 0; l < lay.layers; ++l) {
                    const int nt = lay.nt[l];
                    const uint32_t idesc = idesc_tf32(128, nt);
                    const uint32_t d = tmem + ((l & 1) ? kTpD1 : 0u);
                    for (int c = 0; c < lay.chunks[l]; ++c, ++q) {
                        mbar_wait(&a_ready[c], (aph >> c) & 1u);
                        aph ^= 1u << c;
                        const int st = (int)(q % kMlpStagesT);
                        mbar_wait(&mb_full[st], (q / kMlpStagesT) & 1u);
                        tc_after_sync();
                        const uint32_t bh = smem_u32(ring + (size_t)st * kMlpStageBytes);
                        const uint32_t bl = bh + (uint32_t)nt * kGemmKc * 4;
#pragma unroll
                        for (int s = 0; s < kGemmKc / 8; ++s) {
                            const uint32_t k0 = (uint32_t)(c * kGemmKc + 8 * s);
                            const uint32_t boff = (uint32_t)(2 * s) * kCoreBytes;
                            const uint64_t dbh = umma_desc(bh + boff, kCoreBytes, kGroupBytes);
                            const uint64_t dbl = umma_desc(bl + boff, kCoreBytes, kGroupBytes);
                            mma_tf32_at(d, tmem + kTpA + k0, dbh, idesc, (c > 0 || s > 0) ? 1u : 0u);
                            mma_tf32_at(d, tmem + kTpA + k0, dbl, idesc, 1u);
                            mma_tf32_at(d, tmem + kTpAlo + k0, dbh, idesc, 1u);
                        }
                        mma_commit(&mb_empty[st]);
                    }
                    mma_commit(&mb_layer);
                }
            }
        }
        __syncwarp();
    } else {
        // ---- compute warps: encode, epilogues, staging stores ----
        uint32_t lphase = 0;
        const int ex = 1 + 2 * a.l_x;
        const int kpad0 = lay.chunks[0] * kGemmKc;
        float* S = reinterpret_cast<float*>(smem + (size_t)kMlpStagesT * kMlpStageBytes);  // [128][kStgLd]
        const int r = (warp & 3) * 32 + lane;  // = the TMEM lane this thread may access
        float* srow = S + r * kStgLd;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            const int64_t m0 = (int64_t)tile * 128;
            const int64_t m = m0 + r;
            const bool rv = m < a.n;
            {  // positional encoding -> staging tile (warp group: x, y, z, time + zero padding)
                const int kb = wg * ex;
                if (wg < 3) {
                    const double v = rv ? (double)a.pos[m * a.pos_stride + wg] * a.inv_scale : 0.0;
                    srow[kb] = (float)v;
                    double sn, co;
                    sincospi(v, &sn, &co);
                    for (int l = 0; l < a.l_x; ++l) {
                        if (l) sincospi_double(sn, co);
                        srow[kb + 1 + 2 * l] = (float)sn;
                        srow[kb + 2 + 2 * l] = (float)co;
                    }
                } else {
                    for (int k = kb; k < kpad0; ++k) srow[k] = k - kb < a.te.n ? a.te.v[k - kb] : 0.f;
                }
            }
            bar_compute();
            // A = split(staging) for layer 0, one 32-column chunk per a_ready phase
            for (int c = 0; c < lay.chunks[0]; ++c) {
                const int col = c * 32 + 8 * wg;
                uint32_t hv[8], lv[8];
#pragma unroll
                for (int j = 0; j < 8; j += 4) {
                    const float4 x = *reinterpret_cast<const float4*>(srow + col + j);
                    float h, lo;
                    split_exact(x.x, h, lo); hv[j] = __float_as_uint(h); lv[j] = __float_as_uint(lo);
                    split_exact(x.y, h, lo); hv[j + 1] = __float_as_uint(h); lv[j + 1] = __float_as_uint(lo);
                    split_exact(x.z, h, lo); hv[j + 2] = __float_as_uint(h); lv[j + 2] = __float_as_uint(lo);
                    split_exact(x.w, h, lo); hv[j + 3] = __float_as_uint(h); lv[j + 3] = __float_as_uint(lo);
                }
                tmem_st8(tl + kTpA + (uint32_t)col, hv);
                tmem_st8(tl + kTpAlo + (uint32_t)col, lv);
                tmem_st_wait();
                tc_before_sync();
                __syncwarp();
                if (lane == 0) mbar_arrive(&a_ready[c]);
            }
            for (int l = 0; l < lay.layers; ++l) {
                // the staging tile holds layer l's input: store it for the backward while layer
                // l's MMAs finish
                if (l == 0 && a.X) store_staged(S, a.X, a.ldx, m0, a.n, a.din, nullptr, 0, kMlpThreads / 32);
                if (l > 0 && a.H[l - 1])
                    store_staged(S, a.H[l - 1], a.ldh, m0, a.n, lay.rows[l - 1], a.Hbits[l - 1], 0, kMlpThreads / 32);
                mbar_wait(&mb_layer, lphase & 1u);
                ++lphase;
                bar_compute();  // the staging tile is free again
                tc_after_sync();
                const float* bias = a.params + lay.b_off[l];
                const int rows = lay.rows[l], nt = lay.nt[l];
                const uint32_t dl = (l & 1) ? kTpD1 : 0u;
                if (l + 1 < lay.layers) {
                    // epilogue in the next layer's K chunks: D -> bias, ReLU -> staging + A
                    for (int c = 0; c < lay.chunks[l + 1]; ++c) {
                        const int col = c * 32 + 8 * wg;
                        uint32_t v[8], hv[8], lv[8];
                        float x[8];
                        if (col < nt) {
                            tmem_ld8(tl + dl + (uint32_t)col, v);
#pragma unroll
                            for (int j = 0; j < 8; ++j)
                                x[j] = col + j < rows ? fmaxf(__uint_as_float(v[j]) + __ldg(bias + col + j), 0.f) : 0.f;
                        } else {
#pragma unroll
                            for (int j = 0; j < 8; ++j) x[j] = 0.f;
                        }
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            float h, lo;
                            split_exact(x[j], h, lo);
                            hv[j] = __float_as_uint(h);
                            lv[j] = __float_as_uint(lo);
                        }
                        *reinterpret_cast<float4*>(srow + col) = make_float4(x[0], x[1], x[2], x[3]);
                        *reinterpret_cast<float4*>(srow + col + 4) = make_float4(x[4], x[5], x[6], x[7]);
                        tmem_st8(tl + kTpA + (uint32_t)col, hv);
                        tmem_st8(tl + kTpAlo + (uint32_t)col, lv);
                        tmem_st_wait();
                        tc_before_sync();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&a_ready[c]);
                    }
                    bar_compute();  // the staging tile is complete before it is stored
                } else if (warp < 4) {
                    uint32_t v[16];
                    tmem_ld16(tl + dl, v);
                    if (rv)
#pragma unroll
                        for (int j = 0; j < 16; ++j)
                            if (j < rows) a.out[m * a.out_stride + j] = __uint_as_float(v[j]) + __ldg(bias + j);
                }
            }
            tc_before_sync();
            bar_compute();  // (the next tile's encoding overwrites the staging tile)
        }
    }
    tc_before_sync();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

size_t mlp_tm_smem_bytes() { return (size_t)kMlpStagesT * kMlpStageBytes + (size_t)128 * kStgLd * 4; }

size_t mlp_fused_smem_bytes() { return 2 * (size_t)kMlpAHalf + (size_t)kMlpStages * kMlpStageBytes; }

void launch_pack_weights(const MlpLayout& lay, const float* params, char* out, cudaStream_t st) {
    k_pack_weights<<<dim3(64, lay.layers), 256, 0, st>>>(lay, params, out);
}

void launch_mlp_fwd_fused(const MlpFwdArgs& a, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_mlp_fwd_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mlp_fused_smem_bytes());
        cudaFuncSetAttribute(k_mlp_fwd_tm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mlp_tm_smem_bytes());
        cudaFuncSetAttribute(k_mlp_fwd_tp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mlp_tm_smem_bytes());
        attr = true;
    }
    if (a.n <= 0) return;
    const int ntiles = (int)((a.n + 127) / 128);
    static const bool tmem_a = [] {  // TSB_MLP_ATMEM=0: activations in shared memory (A/B timing; 3.5 vs 2.5 ms)
        const char* e = std::getenv("TSB_MLP_ATMEM");
        return !(e && e[0] == '0');
    }();
    static const bool unpiped = [] {  // TSB_MLP_PIPE=0: layer-serial TMEM kernel (A/B timing)
        const char* e = std::getenv("TSB_MLP_PIPE");
        return e && e[0] == '0';
    }();
    if (tmem_a && !unpiped) {
        k_mlp_fwd_tp<<<std::min(ntiles, 148), kMlpThreadsP, mlp_tm_smem_bytes(), st>>>(a);
        return;
    }
    if (tmem_a) {
        k_mlp_fwd_tm<<<std::min(ntiles, 148), kMlpThreads + 32, mlp_tm_smem_bytes(), st>>>(a);
        return;
    }
    k_mlp_fwd_fused<<<std::min(ntiles, 148), kMlpThreads + 32, mlp_fused_smem_bytes(), st>>>(a);
}

}  // namespace tsb
