// tc_scan.cu — tensor-core (tcgen05) fused distance + top-K' scan, sm_100a.
//
// Same contract as the exact-fp32 scan in knn.cu (replaces the reference's
// _knn_scan_tile / _nn1_scan_tile, /root/reference/pkg/src/parlink/
// neighbors.py:119-160,191-217): one CTA owns 128 query rows for the whole
// (pruned) index sweep and leaves, per row, the K' = 32R best candidates by
// an approximate distance; the float64 refine + certificate in knn.cu makes
// the final result exact.
//
// Numerics.  Both operands are centred on the query block's
// centroid c, scaled by a power of two s and split into two fp16 terms:
//   q~ = hi + lo ~ (q - c) s,  x~ ~ (x - c) s   (relative error 2^-22).
// Three kind::f16 MMAs per 16 dims (hi.hi + hi.lo + lo.hi) give <q~, x~>
// with fp32 accumulation, and the epilogue forms
//   a = |q~|^2 + |x~|^2 - 2<q~, x~>
// with the squared norms of the represented vectors, i.e. the squared
// distance of the represented points up to fp32 rounding.  Centring keeps
// |q~|, |x~| at the scale of the data's local spread instead of its absolute
// position; the split keeps cross-cluster distances (the connect passes)
// resolvable.  The float64 refine certifies every row rigorously.
//
// CTA = 9 warps, warp-specialised:
//   warps 0-3  prep:     A tile once; then per visited index block, centre /
//                        scale / round the 128 points into the canonical
//                        K-major no-swizzle smem layout + their |x^|^2;
//                        warp 0 also runs the pruning visitor.
//   warp  8    MMA:      one elected thread issues tcgen05.mma (M=128,
//                        N=128, K=16) into a TMEM accumulator stage and
//                        tcgen05.commit's it to an mbarrier.
//   warps 4-7  epilogue: tcgen05.ld one accumulator row per thread (thread
//                        = query row), threshold filter (bit mask per 32
//                        columns), branch-free shift-insertion into the
//                        row's 32-entry register list.  No distance tile
//                        ever reaches HBM.
// Two pipeline stages (B tile + TMEM accumulator) overlap prep(t+1), MMA and
// epilogue(t).
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "scan_common.cuh"
#include "tc_scan.cuh"

namespace slk {
namespace tc {

using namespace scan;

constexpr int NTHREADS = 288;
constexpr int NSTAGE = 2;
constexpr uint32_t TMEM_COLS = 256;  // 2 stages x 128 fp32 columns

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void fence_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// Shared-memory matrix descriptor, K-major, no swizzle (canonical layout
// ((8,m),(8,2)) of 16-byte core-matrix rows): LBO = byte distance between the
// two 8-element K halves of one MMA step, SBO = between 8-row groups.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
    return d;                // base offset 0, layout type SWIZZLE_NONE
}

// Instruction descriptor: F32 accumulate, F16 A and B, both K-major, M=128, N=128.
constexpr uint32_t IDESC = (1u << 4) | (0u << 7) | (0u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(IDESC), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
          "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
          "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; i++) v[i] = __uint_as_float(r[i]);
}

// Two-term fp16 split of a centred, scaled pair: v ~ hi + lo with relative
// error <= 2^-22 (lo = fp16(v - hi), v - hi exact in fp32); accumulates the
// squared norm of the represented value hi + lo (exact in fp32) into nrm.
__device__ __forceinline__ void split2(float v0, float v1, __half2 &hi, __half2 &lo, float &nrm) {
    hi = __floats2half2_rn(v0, v1);
    const float2 fh = __half22float2(hi);
    lo = __floats2half2_rn(__fsub_rn(v0, fh.x), __fsub_rn(v1, fh.y));
    const float2 fl = __half22float2(lo);
    const float w0 = __fadd_rn(fh.x, fl.x), w1 = __fadd_rn(fh.y, fl.y);
    nrm = __fmaf_rn(w0, w0, nrm);
    nrm = __fmaf_rn(w1, w1, nrm);
}

// ------------------------------------------------------------- smem plan
struct Plan {
    uint32_t a, b, xx, xcol, qq, cq, misc, bars, total;
};

__host__ __device__ inline Plan make_plan(int dk, int R) {
    Plan p{};
    uint32_t off = 0;
    auto take = [&](uint32_t bytes, uint32_t align) {
        off = (off + align - 1) / align * align;
        uint32_t at = off;
        off += bytes;
        return at;
    };
    const uint32_t tile = (uint32_t)BM * dk * 2;  // 128 rows x dk fp16
    p.a = take(2 * tile, 1024);           // A_hi, A_lo
    p.b = take(2 * tile * NSTAGE, 1024);  // per stage: B_hi, B_lo
    p.xx = take(NSTAGE * BN * 4, 16);
    p.xcol = take(NSTAGE * BN * 4, 16);
    p.qq = take(BM * 4, 16);
    p.cq = take(dk * 4, 16);
    p.misc = take(64, 16);  // part[4] float, next block, stage blocks[2], tmem base
    p.bars = take(8 * 3 * NSTAGE, 8);
    p.total = off;
    return p;
}

struct Misc {
    float part[4];
    int next_blk;
    int stage_blk[NSTAGE];
    uint32_t tmem_base;
};

template <int MODE, int R>
__global__ void __launch_bounds__(NTHREADS, 1) tc_scan_kernel(TcArgs a) {
    extern __shared__ __align__(1024) unsigned char smem[];
    const int dk = a.dk;
    const Plan P = make_plan(dk, R);
    unsigned char *sA = smem + P.a;
    unsigned char *sB = smem + P.b;
    float *s_xx = reinterpret_cast<float *>(smem + P.xx);
    int *s_xcol = reinterpret_cast<int *>(smem + P.xcol);
    float *s_qq = reinterpret_cast<float *>(smem + P.qq);
    float *s_cq = reinterpret_cast<float *>(smem + P.cq);
    Misc *misc = reinterpret_cast<Misc *>(smem + P.misc);
    uint64_t *bfull = reinterpret_cast<uint64_t *>(smem + P.bars);
    uint64_t *tfull = bfull + NSTAGE;
    uint64_t *sfree = tfull + NSTAGE;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t qb = a.qb0 + blockIdx.x;
    const int64_t row_base = qb * BM;
    const int64_t nxb = (a.nx + BN - 1) / BN;
    const uint32_t tile_bytes = (uint32_t)BM * dk * 2;
    const uint32_t sbo = (uint32_t)dk * 16;  // (dk/8) core matrices of 128 B per 8-row group

    // ---- setup: barriers, TMEM, per-row state
    if (tid == 0) {
        for (int s = 0; s < NSTAGE; s++) {
            mbar_init(&bfull[s], 128);
            mbar_init(&tfull[s], 1);
            mbar_init(&sfree[s], 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int i = 0; i < 4; i++) misc->part[i] = INFINITY;
    }
    if (warp == 8) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&misc->tmem_base)),
                     "r"(TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    // s_cq[t] = -c_t * s (exact: s is a power of two), so x^ = fp16(fma(x, s, s_cq[t]))
    for (int t = tid; t < dk; t += NTHREADS)
        s_cq[t] = t < a.d ? -a.qcentroid[(int64_t)t * a.nqb_total + qb] * a.scale : 0.0f;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = misc->tmem_base;

    if (warp < 4) {
        // ===================== prep warps: A once, then B per visited block
        const int r = tid;  // 0..127: query row (A) / index point (B)
        const float sc = a.scale;
        {
            float qq = 0.0f;
            const float *src = a.qp + qb * (int64_t)a.dp * BM + r;
            unsigned char *dst = sA + (r >> 3) * sbo + (r & 7) * 16;
            for (int t0 = 0; t0 < dk; t0 += 8) {
                __half2 h[4], l[4];
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    int t = t0 + 2 * u;
                    float v0 = __fmaf_rn(src[t * BM], sc, s_cq[t]);  // padded dims: 0*s + 0
                    float v1 = __fmaf_rn(src[(t + 1) * BM], sc, s_cq[t + 1]);
                    split2(v0, v1, h[u], l[u], qq);
                }
                *reinterpret_cast<uint4 *>(dst + (t0 >> 3) * 128) = *reinterpret_cast<uint4 *>(h);
                *reinterpret_cast<uint4 *>(dst + tile_bytes + (t0 >> 3) * 128) = *reinterpret_cast<uint4 *>(l);
            }
            s_qq[r] = qq;
        }
        BlockVisitor vis{a.sb_order + (int64_t)blockIdx.x * a.nsb, a.sb_key + (int64_t)blockIdx.x * a.nsb,
                         a.sb_lb + (int64_t)blockIdx.x * a.nsb, a.blk_lb + (int64_t)blockIdx.x * nxb,
                         a.nsb, nxb};
        int64_t computed = 0;
        for (int it = 0;; it++) {
            const int s = it & 1;
            const uint32_t use = (uint32_t)(it >> 1);
            // pruning decision by warp 0, broadcast to the 4 prep warps
            if (warp == 0) {
                volatile float *part = misc->part;
                float thr_max = fmaxf(fmaxf(part[0], part[1]), fmaxf(part[2], part[3])) * a.inv_scale2;
                int64_t jb = vis.next(thr_max, lane);
                if (lane == 0) misc->next_blk = (int)jb;
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");
            const int jb = misc->next_blk;
            asm volatile("bar.sync 2, 128;" ::: "memory");  // next_blk consumed before rewrite
            mbar_wait(&sfree[s], (use & 1) ^ 1);
            if (jb < 0) {
                if (tid == 0) misc->stage_blk[s] = -1;
                mbar_arrive(&bfull[s]);
                break;
            }
            computed++;
            float xx = 0.0f;
            const float *src = a.xp + (int64_t)jb * a.dp * BN + r;
            unsigned char *dst = sB + s * 2 * tile_bytes + (r >> 3) * sbo + (r & 7) * 16;
            for (int t0 = 0; t0 < dk; t0 += 32) {
                // 32 loads in flight per thread, coalesced across the 128 points;
                // dims in [d, dk) are zero in the packed layout
                float v[32];
                const float *col = src + t0 * BN;
                if (t0 + 32 <= dk) {
#pragma unroll
                    for (int u = 0; u < 32; u++) v[u] = __ldg(col + u * BN);
                } else {
#pragma unroll
                    for (int u = 0; u < 16; u++) v[u] = __ldg(col + u * BN);
#pragma unroll
                    for (int u = 16; u < 32; u++) v[u] = 0.0f;
                }
#pragma unroll
                for (int g = 0; g < 4; g++) {
                    if (t0 + g * 8 >= dk) break;
                    __half2 h[4], l[4];
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        const int t = t0 + g * 8 + 2 * u;
                        const float v0 = __fmaf_rn(v[g * 8 + 2 * u], sc, s_cq[t]);
                        const float v1 = __fmaf_rn(v[g * 8 + 2 * u + 1], sc, s_cq[t + 1]);
                        split2(v0, v1, h[u], l[u], xx);
                    }
                    *reinterpret_cast<uint4 *>(dst + ((t0 >> 3) + g) * 128) = *reinterpret_cast<uint4 *>(h);
                    *reinterpret_cast<uint4 *>(dst + tile_bytes + ((t0 >> 3) + g) * 128) = *reinterpret_cast<uint4 *>(l);
                }
            }
            s_xx[s * BN + r] = xx;
            if (MODE == MODE_COLOR) {
                int64_t gj = (int64_t)jb * BN + r;
                s_xcol[s * BN + r] = gj < a.nx ? a.xcolor[gj] : -1;
            }
            if (tid == 0) misc->stage_blk[s] = jb;
            fence_async_smem();  // generic-proxy smem writes → visible to the tensor core
            mbar_arrive(&bfull[s]);
        }
        if (tid == 0 && a.tiles_done) atomicAdd(a.tiles_done, (unsigned long long)computed);
    } else if (warp == 8) {
        // ===================== MMA issuer (one elected thread)
        if (lane == 0) {
            const uint32_t a_base = smem_u32(sA), b_base = smem_u32(sB);
            for (int it = 0;; it++) {
                const int s = it & 1;
                const uint32_t use = (uint32_t)(it >> 1);
                mbar_wait(&bfull[s], use & 1);
                tc_fence_after();
                if (misc->stage_blk[s] < 0) {
                    mbar_arrive(&tfull[s]);
                    break;
                }
                const uint32_t d_tmem = tmem + (uint32_t)s * 128;
                // <q~, x~> = hi.hi + hi.lo + lo.hi (the lo.lo term, <= 2^-22 |q~||x~|, is dropped)
                const uint32_t bs = b_base + s * 2 * tile_bytes;
                for (int k = 0; k < dk / 16; k++) {
                    const uint64_t ah = umma_desc(a_base + k * 256, 128, sbo);
                    const uint64_t al = umma_desc(a_base + tile_bytes + k * 256, 128, sbo);
                    const uint64_t bh = umma_desc(bs + k * 256, 128, sbo);
                    const uint64_t bl = umma_desc(bs + tile_bytes + k * 256, 128, sbo);
                    umma_f16(d_tmem, ah, bh, k > 0 ? 1u : 0u);
                    umma_f16(d_tmem, ah, bl, 1u);
                    umma_f16(d_tmem, al, bh, 1u);
                }
                umma_commit(&tfull[s]);
            }
        }
        __syncwarp();
    } else {
        // ===================== epilogue warps: one query row per thread
        const int ew = warp - 4;  // TMEM lane quarter
        const int row = ew * 32 + lane;
        const int64_t gi = row_base + row;
        // qid (gathered queries): id of the row in the index, -1 for padding
        const int64_t self_id = (gi < a.nq && a.qid) ? (int64_t)a.qid[gi] : gi;
        const bool row_ok = gi < a.nq && self_id >= 0;
        float qq = 0.0f;  // |q^|^2, written by the prep warps: read after the first tfull
        const int qc = (MODE == MODE_COLOR && row_ok) ? a.qcolor[gi] : -1;
        // This thread's row keeps its 32 best (approximate value, id) pairs in
        // registers, ascending; thr = the 32nd.  Ties may be ordered either
        // way: the certificate only needs every dropped candidate >= thr.
        float lv[32];
        int li[32];
#pragma unroll
        for (int p = 0; p < 32; p++) {
            lv[p] = INFINITY;
            li[p] = -1;
        }
        float thr = INFINITY;

        for (int it = 0;; it++) {
            const int s = it & 1;
            const uint32_t use = (uint32_t)(it >> 1);
            mbar_wait(&tfull[s], use & 1);
            tc_fence_after();
            // bfull (prep done with A and this B) happened before tfull
            if (it == 0) qq = s_qq[row];
            const int jb = misc->stage_blk[s];
            if (jb < 0) break;
            const int64_t col0 = (int64_t)jb * BN;
            const uint32_t taddr = tmem + ((uint32_t)(ew * 32) << 16) + (uint32_t)s * 128;
            // columns this row may take from this block: inside the index, not
            // itself (32-bit, once per tile instead of 64-bit math per value)
            const int64_t rem = a.nx - col0;
            const int col_limit = row_ok ? (rem < BN ? (int)rem : BN) : 0;
            const int self_col =
                (MODE == MODE_SELF && self_id >= col0 && self_id < col0 + BN) ? (int)(self_id - col0) : -1;
            const float *xxs = s_xx + s * BN;
#pragma unroll 1
            for (int c0 = 0; c0 < BN; c0 += 32) {
                float dot[32];
                tmem_ld32(taddr + c0, dot);
                uint32_t valid = c0 >= col_limit ? 0u : (col_limit - c0 >= 32 ? 0xffffffffu : ((1u << (col_limit - c0)) - 1u));
                if (self_col >= c0 && self_col < c0 + 32) valid &= ~(1u << (self_col - c0));
                uint32_t pass = 0;
                float av[32];
#pragma unroll
                for (int i = 0; i < 32; i += 4) {
                    const float4 x4 = *reinterpret_cast<const float4 *>(xxs + c0 + i);
                    av[i + 0] = __fmaf_rn(-2.0f, dot[i + 0], __fadd_rn(qq, x4.x));
                    av[i + 1] = __fmaf_rn(-2.0f, dot[i + 1], __fadd_rn(qq, x4.y));
                    av[i + 2] = __fmaf_rn(-2.0f, dot[i + 2], __fadd_rn(qq, x4.z));
                    av[i + 3] = __fmaf_rn(-2.0f, dot[i + 3], __fadd_rn(qq, x4.w));
                    pass |= (av[i + 0] < thr ? 1u : 0u) << (i + 0);
                    pass |= (av[i + 1] < thr ? 1u : 0u) << (i + 1);
                    pass |= (av[i + 2] < thr ? 1u : 0u) << (i + 2);
                    pass |= (av[i + 3] < thr ? 1u : 0u) << (i + 3);
                }
                pass &= valid;
                if (MODE == MODE_COLOR && pass) {
#pragma unroll
                    for (int i = 0; i < 32; i++)
                        if (s_xcol[s * BN + c0 + i] == qc) pass &= ~(1u << i);
                }
                if (MODE == MODE_MASK && pass) {
                    for (int i = 0; i < 32; i++)
                        if (((pass >> i) & 1u) && a.mask[gi * a.nx + col0 + c0 + i] == 0) pass &= ~(1u << i);
                }
                while (pass) {
                    const int i = __ffs(pass) - 1;
                    pass &= pass - 1;
                    float v = av[0];
#pragma unroll
                    for (int u = 1; u < 32; u++) v = (i == u) ? av[u] : v;
                    if (!(v < thr)) continue;  // the threshold may have dropped
                    const int id = (int)(col0 + c0 + i);
                    // shift-insert: new[p] = v < old[p-1] ? old[p-1] : (v < old[p] ? v : old[p])
                    bool c_next = v < lv[31];
#pragma unroll
                    for (int p = 31; p > 0; p--) {
                        const bool c_prev = v < lv[p - 1];
                        lv[p] = c_prev ? lv[p - 1] : (c_next ? v : lv[p]);
                        li[p] = c_prev ? li[p - 1] : (c_next ? id : li[p]);
                        c_next = c_prev;
                    }
                    if (c_next) {
                        lv[0] = v;
                        li[0] = id;
                    }
                    thr = lv[31];
                }
            }
            tc_fence_before();
            mbar_arrive(&sfree[s]);  // TMEM stage, B tile and xx of stage s are free
            float wm = row_ok ? thr : -INFINITY;
            for (int o = 16; o; o >>= 1) wm = fmaxf(wm, __shfl_xor_sync(FULL, wm, o));
            if (lane == 0) ((volatile float *)misc->part)[ew] = wm;
        }
        // write this row's candidate list
        if (gi >= a.row0 && gi < a.row1 && row_ok) {
            int32_t *dst = a.cand + (gi - a.row0) * 32;
#pragma unroll
            for (int q = 0; q < 32; q++) dst[q] = li[q];
            a.kth[gi - a.row0] = li[31] >= 0 ? lv[31] : INFINITY;
            a.qhat[gi - a.row0] = qq;
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 8) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS)
                     : "memory");
    }
}

template <int MODE, int R>
void launch_mode(const TcArgs &args, int64_t nqb, cudaStream_t s) {
    const Plan P = make_plan(args.dk, R);
    SLK_CUDA(cudaFuncSetAttribute(tc_scan_kernel<MODE, R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)P.total));
    tc_scan_kernel<MODE, R><<<(unsigned)nqb, NTHREADS, P.total, s>>>(args);
    SLK_CHECK_LAUNCH();
}

template <int R>
void launch_r(int mode, const TcArgs &args, int64_t nqb, cudaStream_t s) {
    switch (mode) {
        case MODE_NONE: launch_mode<MODE_NONE, R>(args, nqb, s); break;
        case MODE_MASK: launch_mode<MODE_MASK, R>(args, nqb, s); break;
        case MODE_COLOR: launch_mode<MODE_COLOR, R>(args, nqb, s); break;
        default: launch_mode<MODE_SELF, R>(args, nqb, s); break;
    }
}

size_t smem_bytes(int d, int R) { return make_plan(((d + 15) / 16) * 16, R).total; }

// Register lists hold K' = 32 candidates: the tensor path serves k <= 31.
bool supported(int d, int R) { return R == 1 && d <= 256 && smem_bytes(d, R) <= 227 * 1024; }

void launch(int mode, int R, const TcArgs &args, int64_t nqb, cudaStream_t s) {
    (void)R;
    launch_r<1>(mode, args, nqb, s);
}

}  // namespace tc
}  // namespace slk
