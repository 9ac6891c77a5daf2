// tc_scan.cu — tensor-core (tcgen05) fused distance + top-K' scan, sm_100a.
//
// Same contract as the exact-fp32 scan in knn.cu (replaces the reference's
// _knn_scan_tile / _nn1_scan_tile, /root/reference/pkg/src/parlink/
// neighbors.py:119-160,191-217): one CTA owns 128 query rows for the whole
// (pruned) index sweep and leaves, per row, the K' best candidates by an
// approximate distance; the float64 refine + certificate in knn.cu makes the
// final result exact.
//
// Numerics.  Both operands are centred on the query block's
// centroid c, scaled by a power of two s and split into two fp16 terms:
//   q~ = hi + lo ~ (q - c) s,  x~ ~ (x - c) s   (relative error 2^-22).
// Three kind::f16 MMAs per 16 dims (hi.hi + hi.lo + lo.hi) give <q~, x~>
// with fp32 accumulation; the epilogue forms b = |x~|^2 - 2<q~,x~> and the
// row constant |q~|^2 is added once per row (a = |q~|^2 + b).  Centring keeps
// |q~|, |x~| at the scale of the data's local spread; the split keeps
// cross-cluster distances (the connect passes) resolvable.
//
// Operand staging.  The index is stored once per call in a "tc-packed" fp32
// layout (tcpack_kernel in knn.cu): block jb is one contiguous 128 x dk x 4 B
// run whose bytes sit exactly where the converted fp16 hi/lo UMMA tiles of
// the same points go (point r, dims 8g..8g+3 at the hi core-matrix row of
// (r, g), dims 8g+4..8g+7 at the lo one).  A block therefore arrives with
// ONE cp.async.bulk (TMA bulk copy, mbarrier complete_tx) and is converted
// in place, each thread touching only its own point's bytes.
//
// CTA = 14 warps, warp-specialised, all hand-offs on mbarriers:
//   warp  9    producer: walks the pruned visit order (32 superblocks per
//              step, ballots), issues the bulk copies of raw blocks (and their
//              colours) into a ring of NB stages, NB - 1 blocks ahead.
//   warps 0-3, 10-13  convert: centre / scale / split the stage in place into
//              the canonical K-major no-swizzle layout + |x~|^2 per point (two
//              threads per point, one per half of the dims).
//   warp  8    MMA:      one elected thread issues tcgen05.mma (M=128, N=128,
//              K=16) into one of NT TMEM accumulator stages, then commits to
//              the stage's "B empty" and the accumulator's "full" barriers.
//   warps 4-7  epilogue: tcgen05.ld one accumulator row per thread (thread =
//              query row), chunk minimum vs the row threshold (fast path), and
//              only for chunks with a hit: exact pass mask, staging of the 32
//              values in smem, shift-insertion into the row's K'-entry
//              register list.  No distance tile ever reaches HBM.
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "common.cuh"
#include "scan_common.cuh"
#include "tc_scan.cuh"

namespace slk {
namespace tc {
namespace {

using namespace scan;

#include "tc_ptx.cuh"  // PTX wrappers (inside this namespace)

// ------------------------------------------------------------- smem plan
// (Measured at C3/C5: 4 convert warps with 157 registers and 32-column
// epilogue steps beat 8 convert warps capped at 128 registers.)
// QB query blocks per CTA share every converted index tile (QB = 2 halves the
// conversion work per query row; its 8 epilogue warps cap registers at 128,
// so it serves K' <= 16).  Warps: convert 0-3, epilogue 4 .. 4+4QB-1, then
// MMA, then producer.
template <int QB> struct Cfg {
    static constexpr int NTHREADS = 192 + 128 * QB;
    static constexpr int WARP_MMA = 4 + 4 * QB;
    static constexpr int WARP_PROD = 5 + 4 * QB;
    static constexpr int NT = 4 / QB;  // TMEM accumulator stages of 128 QB columns: 512 columns
};
constexpr int NTMAX = 4;
constexpr int MAX_NB = 6;    // B operand stages
constexpr int NMETA = MAX_NB + NTMAX;  // per-tile metadata ring (see producer)
constexpr uint32_t TMEM_COLS = 512;
constexpr int CH = 32;  // accumulator columns per epilogue step (tcgen05.ld .x32)
constexpr uint32_t CH_ALL = 0xffffffffu;
// Augmented K: one extra 16-column K step carries the norm term, in small
// separate tiles (128 rows x 16 fp16, hi only) so the bulk copies move only
// the real dims.  A: columns 0, 1 = 2^14; B: columns 0, 1 = two-term fp16
// split of -|x~|^2 2^-15.  One extra hi.hi MMA adds -|x~|^2 / 2 to the
// accumulator, so the epilogue reads acc = <q~,x~> - |x~|^2 / 2 = -b / 2
// directly (knn.cu:tensor_scale keeps |x~|^2 2^-15 below the fp16 range).
constexpr uint32_t AUG_TILE = BM * 16 * 2;  // bytes; canonical layout, SBO = 256
constexpr float NORM_A = 16384.0f;       // 2^14
constexpr float NORM_B_SCALE = -0x1p-15f;
constexpr int STG_STRIDE = CH + 4;  // per-row chunk staging (CH + 4 floats: conflict-free STS.128)
constexpr uint32_t SMEM_LIMIT = 227 * 1024;

struct Plan {
    uint32_t a, b, aaug, baug, xx, xcol, qq, cq, stg, misc, bars, total;
    int nb;  // B stages that fit
};

// Large d (chunked kernel, CK): the query tile's hi term lives in TMEM
// columns [A_COL, A_COL + dk/2), its lo term in shared memory, and the index
// blocks stream in KC-dim chunks (tcpack stores each block as dk/KC
// consecutive KC-dim sub-blocks), so d up to CK_MAX_DK fits.  Two
// accumulator stages (columns 0-255).
constexpr int KC = 32;
constexpr int CK_MAX_DK = 512;
constexpr uint32_t A_COL = 256;

// aug: the norm rides in the augmented K step (no |x~|^2 array); kc > 0: the
// chunked large-d layout (A = lo term only, B stages of kc dims)
__host__ __device__ inline Plan make_plan(int dk, bool aug, int qb, int kc = 0, int ew = 0) {
    Plan p{};
    uint32_t off = 0;
    auto take = [&](uint32_t bytes, uint32_t align) {
        off = (off + align - 1) / align * align;
        uint32_t at = off;
        off += bytes;
        return at;
    };
    const uint32_t stage = (uint32_t)BM * (kc > 0 ? kc : dk) * 4;  // hi + lo fp16 tiles = raw fp32 block
    p.a = take(kc > 0 ? (uint32_t)BM * dk * 2 : stage * qb, 1024);
    p.aaug = aug ? take(AUG_TILE, 1024) : 0u;
    p.xx = aug ? 0u : take(NMETA * BN * 4, 16);
    p.xcol = take(NMETA * BN * 4, 16);
    p.qq = take(qb * BM * 4, 16);
    p.cq = take(dk * 4, 16);
    p.stg = take((ew > 0 ? ew : qb) * BM * STG_STRIDE * 4, 16);
    p.misc = take(128, 16);
    p.bars = take(8 * (4 * MAX_NB + 2 * NTMAX + 1), 8);
    off = (off + 1023) / 1024 * 1024;
    const uint32_t per = stage + (aug ? AUG_TILE : 0u);
    int nb = off >= SMEM_LIMIT ? 0 : (int)((SMEM_LIMIT - off) / per);
    p.nb = nb > MAX_NB ? MAX_NB : nb;
    p.b = take(stage * (p.nb > 0 ? p.nb : 0), 1024);
    p.baug = aug ? take(AUG_TILE * (p.nb > 0 ? p.nb : 0), 1024) : 0u;
    p.total = off;
    return p;
}

// position in a ring of n stages and the mbarrier phase parity of the lap
struct Ring {
    int s;
    uint32_t ph;
    int n;
    __device__ __forceinline__ void next() {
        if (++s == n) {
            s = 0;
            ph ^= 1u;
        }
    }
};

struct Misc {
    float part[8];            // per epilogue warp: largest row threshold (a units)
    uint32_t tmem_base;
    int meta_blk[NMETA];      // block id of tile t at slot t % NMETA (-1 = end)
#ifdef SLK_WATCHDOG
    int dbg[4];               // last tile reached by producer / convert / epilogue / MMA
#endif
};

#ifdef SLK_WATCHDOG
__device__ void watchdog_dump(int tag, int it, uint32_t parity, unsigned long long st) {
    extern __shared__ __align__(1024) unsigned char smem[];
    const Plan P = make_plan(64, true);
    const Misc *m = reinterpret_cast<const Misc *>(smem + P.misc);
    const unsigned long long *bars = reinterpret_cast<const unsigned long long *>(smem + P.bars);
    printf("watchdog: block %d thread %d tag %d it %d parity %u state %llx dbg %d %d %d %d "
           "raw %llx %llx %llx %llx %llx\n",
           blockIdx.x, threadIdx.x, tag, it, parity, st, m->dbg[0], m->dbg[1], m->dbg[2], m->dbg[3], bars[0],
           bars[1], bars[2], bars[3], bars[4]);
}
#endif

// Converts the dkm dims (core-matrix columns [0, dkm/8)) of point r of a
// 128-point operand tile in place (raw tc-packed fp32 -> fp16 hi/lo canonical
// layout, K extent dk = dkm) and returns |v|^2 of the unsplit values.
__device__ __forceinline__ float convert_tile(unsigned char *tile, int r, int dkm, int dk, float sc,
                                              const float *s_cq, bool one = false) {
    const uint32_t half_bytes = (uint32_t)BM * dk * 2;
    unsigned char *row = tile + (r >> 3) * (dk * 16) + (r & 7) * 16;
    // four independent partial norms: the accumulation chain would otherwise
    // serialise the conversion (the error bound does not depend on order)
    float nrm4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll 4
    for (int g = 0; g < dkm / 8; g++) {
        float4 *ph = reinterpret_cast<float4 *>(row + g * 128);
        float4 *pl = reinterpret_cast<float4 *>(row + half_bytes + g * 128);
        const float4 u = *ph, w = *pl;
        const float4 c0 = *reinterpret_cast<const float4 *>(s_cq + 8 * g);
        const float4 c1 = *reinterpret_cast<const float4 *>(s_cq + 8 * g + 4);
        const float v[8] = {__fmaf_rn(u.x, sc, c0.x), __fmaf_rn(u.y, sc, c0.y), __fmaf_rn(u.z, sc, c0.z),
                            __fmaf_rn(u.w, sc, c0.w), __fmaf_rn(w.x, sc, c1.x), __fmaf_rn(w.y, sc, c1.y),
                            __fmaf_rn(w.z, sc, c1.z), __fmaf_rn(w.w, sc, c1.w)};
        __half2 h[4], l[4];
        if (one) {
            // one-product scan: the hi term only (the lo tile is never read)
#pragma unroll
            for (int q = 0; q < 4; q++) {
                h[q] = __floats2half2_rn(v[2 * q], v[2 * q + 1]);
                nrm4[q] = __fmaf_rn(v[2 * q], v[2 * q], nrm4[q]);
                nrm4[q] = __fmaf_rn(v[2 * q + 1], v[2 * q + 1], nrm4[q]);
            }
            *reinterpret_cast<uint4 *>(ph) = *reinterpret_cast<uint4 *>(h);
        } else {
#pragma unroll
            for (int q = 0; q < 4; q++) split2(v[2 * q], v[2 * q + 1], h[q], l[q], nrm4[q]);
            *reinterpret_cast<uint4 *>(ph) = *reinterpret_cast<uint4 *>(h);
            *reinterpret_cast<uint4 *>(pl) = *reinterpret_cast<uint4 *>(l);
        }
    }
    return __fadd_rn(__fadd_rn(nrm4[0], nrm4[1]), __fadd_rn(nrm4[2], nrm4[3]));
}

// Writes columns 0, 1 of point r's row of an augmented-step tile (the other
// 14 columns are zeroed once per CTA).
__device__ __forceinline__ void put_norm_terms(unsigned char *aug, int r, float t0, float t1) {
    *reinterpret_cast<__half2 *>(aug + (r >> 3) * 256 + (r & 7) * 16) = __floats2half2_rn(t0, t1);
}

// -|x~|^2 2^-15 as hi + lo fp16 (|hi + lo - v| <= 2^-22 |v| + 2^-25)
__device__ __forceinline__ void norm_split(float xx, float &t0, float &t1) {
    const float v = xx * NORM_B_SCALE;  // exact: power of two
    const float hi = __half2float(__float2half_rn(v));
    t0 = hi;
    t1 = __fsub_rn(v, hi);
}

// Converts query row r of block qb for the chunked kernel straight from the
// tc-packed global copy: the hi term goes to TMEM lane r (columns A_COL +
// dims / 2), the lo term to the shared-memory A tile (canonical K-major,
// SBO = dk * 16).  Returns |q~|^2 of the unsplit values.
__device__ __forceinline__ float convert_query_ck(const float *qblk, unsigned char *sA, int r, int dk, float sc,
                                                  const float *s_cq, uint32_t tmem_lane) {
    float nrm4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    for (int b64 = 0; b64 < dk / 64; b64++) {
        uint32_t hreg[32];
#pragma unroll
        for (int gg = 0; gg < 8; gg++) {
            const int t0 = b64 * 64 + gg * 8;  // first dim of the 8-dim group
            const int c = t0 / KC, g = (t0 % KC) >> 3;
            const float *hp = qblk + (int64_t)c * BM * KC + (r >> 3) * (KC * 4) + g * 32 + (r & 7) * 4;
            const float4 u = *reinterpret_cast<const float4 *>(hp);
            const float4 w = *reinterpret_cast<const float4 *>(hp + BM * KC / 2);
            const float4 c0 = *reinterpret_cast<const float4 *>(s_cq + t0);
            const float4 c1 = *reinterpret_cast<const float4 *>(s_cq + t0 + 4);
            const float v[8] = {__fmaf_rn(u.x, sc, c0.x), __fmaf_rn(u.y, sc, c0.y), __fmaf_rn(u.z, sc, c0.z),
                                __fmaf_rn(u.w, sc, c0.w), __fmaf_rn(w.x, sc, c1.x), __fmaf_rn(w.y, sc, c1.y),
                                __fmaf_rn(w.z, sc, c1.z), __fmaf_rn(w.w, sc, c1.w)};
            __half2 h[4], l[4];
#pragma unroll
            for (int q = 0; q < 4; q++) {
                split2(v[2 * q], v[2 * q + 1], h[q], l[q], nrm4[q]);
                hreg[gg * 4 + q] = *reinterpret_cast<uint32_t *>(&h[q]);
            }
            *reinterpret_cast<uint4 *>(sA + (r >> 3) * (dk * 16) + (t0 >> 3) * 128 + (r & 7) * 16) =
                *reinterpret_cast<uint4 *>(l);
        }
        tmem_st32(tmem_lane + A_COL + (uint32_t)b64 * 32, hreg);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    return __fadd_rn(__fadd_rn(nrm4[0], nrm4[1]), __fadd_rn(nrm4[2], nrm4[3]));
}

// CK: chunked large-d variant (QB = 1, no augmented step): every index block
// arrives as dk / KC stages of KC dims that accumulate into one TMEM stage.
// HS = 2 (QB = 1): two epilogue warps per TMEM lane quarter, each keeping its
// own K' list over one half of every tile's columns (written out as two
// splits that the refine unites, like nsplit): twice the epilogue warps to
// hide the insertion latency of the k-NN pass.
template <int MODE, int KP, bool AUG, int QB, bool CK, int HS = 1>
__global__ void __launch_bounds__(Cfg<QB * HS>::NTHREADS, 1) tc_scan_kernel(TcArgs a) {
    extern __shared__ __align__(1024) unsigned char smem[];
    static_assert(!CK || (QB == 1 && !AUG), "chunked kernel: single query block, norms via smem");
    static_assert(HS == 1 || QB == 1, "column halves only with one query block per CTA");
    constexpr int EW = QB * HS;  // epilogue warp groups (of 4)
    constexpr int NTHREADS = Cfg<EW>::NTHREADS, NT = CK ? 2 : Cfg<QB>::NT;
    const int dk = a.dk;
    const int kc = CK ? KC : dk;  // dims per B stage
    const int nck = dk / kc;      // stages per index block
    const Plan P = make_plan(dk, AUG, QB, CK ? KC : 0, EW);
    float *s_xx = reinterpret_cast<float *>(smem + P.xx);  // !AUG: |x~|^2 per meta slot
    const int nb = P.nb;
    unsigned char *sA = smem + P.a;
    unsigned char *sB = smem + P.b;
    int *s_xcol = reinterpret_cast<int *>(smem + P.xcol);
    float *s_qq = reinterpret_cast<float *>(smem + P.qq);
    float *s_cq = reinterpret_cast<float *>(smem + P.cq);
    float *s_stg = reinterpret_cast<float *>(smem + P.stg);
    Misc *misc = reinterpret_cast<Misc *>(smem + P.misc);
    uint64_t *rawfull = reinterpret_cast<uint64_t *>(smem + P.bars);  // producer -> convert
    uint64_t *bfull = rawfull + MAX_NB;                                 // convert -> MMA
    uint64_t *bempty = bfull + MAX_NB;                                  // MMA commit -> producer
    uint64_t *tfull = bempty + MAX_NB;                                  // MMA commit -> epilogue
    uint64_t *tempty = tfull + NT;                                      // epilogue -> MMA
    uint64_t *afull = tempty + NT;                                      // A tile landed

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t qbl = blockIdx.x / a.nsplit;  // query group (QB blocks) within the launch
    const int split = blockIdx.x - (int)qbl * a.nsplit;
    const int64_t qb = a.qb0 + qbl * QB;        // first query block of the group
    const int nqa = (int)min((int64_t)QB, a.nqb_total - qb);  // query blocks present
    const int64_t nxb = (a.nx + BN - 1) / BN;
    const uint32_t stage_bytes = (uint32_t)BM * kc * 4;
    const uint32_t half_bytes = (uint32_t)BM * kc * 2;
    const uint32_t sbo = (uint32_t)kc * 16;  // (kc/8) core matrices of 128 B per 8-row group
    const int dkm = dk;                      // dims (d rounded up to 16); the norm step is separate
    unsigned char *sAaug = smem + P.aaug;    // AUG: norm-step tiles of A and of each B stage
    unsigned char *sBaug = smem + P.baug;
    const bool one = a.nprod == 1;    // one fp16 product per 16 dims (hi.hi)

    // ---- setup: barriers, TMEM, centring constants
    if (tid == 0) {
        for (int s = 0; s < MAX_NB; s++) {
            mbar_init(&rawfull[s], 1);
            mbar_init(&bfull[s], 128);
            mbar_init(&bempty[s], 1);
        }
        for (int s = 0; s < NT; s++) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], 128 * EW);
        }
        mbar_init(afull, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int i = 0; i < 8; i++) misc->part[i] = INFINITY;
    }
    if (warp == Cfg<EW>::WARP_MMA) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&misc->tmem_base)),
                     "r"(TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    // s_cq[t] = -c_t * s (exact: s is a power of two), so x~ = fma(x, s, s_cq[t])
    for (int t = tid; t < dk; t += NTHREADS)
        s_cq[t] = t < a.d ? -a.gcentroid[(int64_t)t * a.ngroups + qbl] * a.scale : 0.0f;
    if (AUG) {
        // norm-step tiles: columns 2..15 stay zero (columns 0, 1 written per tile)
        for (uint32_t e = tid; e < AUG_TILE / 16; e += NTHREADS)
            reinterpret_cast<uint4 *>(sAaug)[e] = make_uint4(0u, 0u, 0u, 0u);
        for (uint32_t e = tid; e < AUG_TILE * nb / 16; e += NTHREADS)
            reinterpret_cast<uint4 *>(sBaug)[e] = make_uint4(0u, 0u, 0u, 0u);
        fence_async_smem();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = misc->tmem_base;

    if (warp == Cfg<EW>::WARP_PROD) {
        // ===================== producer: visit order + bulk copies
        if (lane == 0 && !CK) {
            mbar_expect_tx(afull, stage_bytes * nqa);
            for (int q = 0; q < nqa; q++)
                bulk_g2s(sA + q * stage_bytes, a.qp + (qb + q) * (int64_t)dk * BM, stage_bytes, afull);
        }
        BlockVisitor vis(a.sb_order + qbl * a.nsb, a.sb_lb + qbl * a.nsb, a.flat_lb + qbl * a.nsb * 32,
                         a.nvalid[qbl], lane, split, a.nsplit);
        int64_t computed = 0;
        Ring rg{0, 0u, nb};  // B stage ring (nck stages per index block)
        for (int it = 0;; it++) {
            // the epilogue warps publish their largest row threshold with an
            // atomic exchange and lane 0 reads them atomically: thresholds only
            // shrink, so any value read is a valid (conservative) bound
            float thr = 0.0f;
            if (lane == 0) {
                float *part = misc->part;
                thr = fmaxf(fmaxf(atomicAdd(&part[0], 0.0f), atomicAdd(&part[1], 0.0f)),
                            fmaxf(atomicAdd(&part[2], 0.0f), atomicAdd(&part[3], 0.0f)));
                if (EW == 2)
                    thr = fmaxf(thr, fmaxf(fmaxf(atomicAdd(&part[4], 0.0f), atomicAdd(&part[5], 0.0f)),
                                           fmaxf(atomicAdd(&part[6], 0.0f), atomicAdd(&part[7], 0.0f))));
                thr *= a.inv_scale2;
            }
            // the visitor's control flow must be warp-uniform
            thr = __shfl_sync(FULL, thr, 0);
            const int64_t jb = vis.next(thr, lane);
#ifdef SLK_WATCHDOG
            if (lane == 0) misc->dbg[0] = it * 100000 + (int)(jb < 0 ? 99999 : jb % 100000);
#endif
            if (lane == 0) {
                // the end marker is one stage; a block is nck stages
                TL(0, it);
                for (int c = 0; c < (jb < 0 ? 1 : nck); c++, rg.next()) {
                    const int s = rg.s;
                    const uint32_t ph = rg.ph;
                    mbar_wait(&bempty[s], ph ^ 1u, 1, it);
                    if (c == 0) TL(1, it);
                    if (c == 0) misc->meta_blk[it % NMETA] = (int)jb;
                    if (jb < 0) {
                        mbar_arrive(&rawfull[s]);
                    } else {
                        // MODE_SELF with xcolor: re-blocked index whose pad entries are marked < 0
                        const bool col = (MODE == MODE_COLOR || (MODE == MODE_SELF && a.xcolor)) && c == 0;
                        mbar_expect_tx(&rawfull[s], stage_bytes + (col ? BN * 4 : 0));
                        bulk_g2s(sB + (size_t)s * stage_bytes, a.xp + (jb * nck + c) * (int64_t)kc * BN,
                                 stage_bytes, &rawfull[s]);
                        if (col)
                            bulk_g2s(s_xcol + (it % NMETA) * BN, a.xcolor + jb * BN, BN * 4, &rawfull[s]);
                    }
                }
                TL(2, it);
                if (jb >= 0) computed++;
            }
            if (jb < 0) break;
        }
        if (lane == 0 && a.tiles_done) atomicAdd(a.tiles_done, (unsigned long long)computed);
    } else if (warp < 4) {
        // ===================== convert warps: A once, then every B stage in place
        const int r = tid;  // 0..127: query row (A) / index point (B)
        const float sc = a.scale;
        if (CK) {
            s_qq[r] = convert_query_ck(a.qp + qb * (int64_t)dk * BM, sA, r, dk, sc, s_cq,
                                       tmem + ((uint32_t)(warp * 32) << 16));
            tc_fence_before();  // published to the MMA warp by the first bfull arrive
        } else {
            mbar_wait(afull, 0, 2, 0);
#pragma unroll
            for (int q = 0; q < QB; q++) {
                // a missing second block (odd count) converts stale smem: its rows are never output
                s_qq[q * BM + r] = convert_tile(sA + q * stage_bytes, r, dkm, dk, sc, s_cq, one);
                if (AUG && q == 0) put_norm_terms(sAaug, r, NORM_A, NORM_A);  // shared by the group
            }
        }
        Ring rg{0, 0u, nb};
        for (int it = 0;; it++) {
            float xx = 0.0f;
            bool end = false;
            for (int c = 0; c < nck; c++, rg.next()) {
                const int s = rg.s;
                const uint32_t ph = rg.ph;
                mbar_wait(&rawfull[s], ph, 3, it);
                if (r == 0 && c == 0) TL(3, it);
                const int jb = misc->meta_blk[it % NMETA];
#ifdef SLK_WATCHDOG
                if (r == 100) misc->dbg[1] = it * 100000 + (jb < 0 ? 99999 : jb % 100000);
#endif
                if (jb < 0) {
                    mbar_arrive(&bfull[s]);
                    end = true;
                    break;
                }
                unsigned char *tile = sB + (size_t)s * stage_bytes;
                xx = __fadd_rn(xx, convert_tile(tile, r, kc, kc, sc, s_cq + c * kc, one));
                if (c == nck - 1) {
                    if (AUG) {
                        float t0, t1;
                        norm_split(xx, t0, t1);
                        put_norm_terms(sBaug + (size_t)s * AUG_TILE, r, t0, t1);
                    } else {
                        s_xx[(it % NMETA) * BN + r] = xx;
                    }
                }
                fence_async_smem();  // generic-proxy smem writes -> visible to the tensor core
                mbar_arrive(&bfull[s]);  // every thread arrives: its writes are released by its own arrive
                if (r == 0 && c == nck - 1) TL(4, it);
            }
            if (end) break;
        }
    } else if (warp == Cfg<EW>::WARP_MMA) {
        // ===================== MMA issuer (the whole warp; elect.sync issues)
        {
            const uint32_t a_base = smem_u32(sA), b_base = smem_u32(sB);
            // descriptors advance by 256 B (one 16-dim K step) = 16 in the
            // address field (bits 0-13, addr >> 4; shared addresses < 2^18)
            const uint64_t aug_a = umma_desc(smem_u32(sAaug), 128, 256);
            Ring rg{0, 0u, nb};
            for (int it = 0;; it++) {
                const int ts = it % NT;
                const uint32_t tph = (uint32_t)(it / NT) & 1u;
                bool end = false;
                for (int c = 0; c < nck; c++, rg.next()) {
                const int s = rg.s;
                const uint32_t ph = rg.ph;
                if (c == 0) TL(5, it);
                mbar_wait(&bfull[s], ph, 4, it);
#ifdef SLK_WATCHDOG
                misc->dbg[3] = it;
#endif
                if (c == 0) {
                    TL(6, it);
                    // the accumulator stage must be drained even for the end marker:
                    // two completions of tfull[ts] ahead of the epilogue would alias
                    // its phase parity
                    mbar_wait(&tempty[ts], tph ^ 1u, 5, it);
                    TL(7, it);
                    if (misc->meta_blk[it % NMETA] < 0) {
                        if (lane == 0) mbar_arrive(&tfull[ts]);
                        end = true;
                        break;
                    }
                }
                tc_fence_after();
                const uint32_t bs = b_base + s * stage_bytes;
                if (CK) {
                    // <q~, x~> over this chunk's K steps: hi from TMEM, lo from smem
                    const uint32_t d_tmem = tmem + (uint32_t)ts * 128;
                    const int kg0 = c * (kc / 16);
                    const uint64_t al0 = umma_desc(a_base + kg0 * 256, 128, (uint32_t)dk * 16);
                    const uint64_t bh0 = umma_desc(bs, 128, sbo);
                    const uint64_t bl0 = umma_desc(bs + half_bytes, 128, sbo);
#pragma unroll 2
                    for (int k = 0; k < kc / 16; k++) {
                        const uint32_t ta = tmem + A_COL + (uint32_t)(kg0 + k) * 8;
                        umma_f16_ta_w(d_tmem, ta, bh0 + 16u * k, (kg0 + k) > 0 ? 1u : 0u);
                        if (!one) {
                            umma_f16_ta_w(d_tmem, ta, bl0 + 16u * k, 1u);
                            umma_f16_w(d_tmem, al0 + 16u * k, bh0 + 16u * k, 1u);
                        }
                    }
                } else {
                const uint64_t bh0 = umma_desc(bs, 128, sbo);
                const uint64_t bl0 = umma_desc(bs + half_bytes, 128, sbo);
                const uint64_t aug_b = umma_desc(smem_u32(sBaug) + s * AUG_TILE, 128, 256);
#pragma unroll
                for (int q = 0; q < QB; q++) {
                    const uint32_t d_tmem = tmem + (uint32_t)(ts * QB + q) * 128;
                    const uint32_t aq = a_base + q * stage_bytes;
                    const uint64_t ah0 = umma_desc(aq, 128, sbo);
                    const uint64_t al0 = umma_desc(aq + half_bytes, 128, sbo);
                    // <q~, x~> = hi.hi + hi.lo + lo.hi (the lo.lo term, <= 2^-22 |q~||x~|, is dropped)
#pragma unroll 4
                    for (int k = 0; k < dkm / 16; k++) {
                        umma_f16_w(d_tmem, ah0 + 16u * k, bh0 + 16u * k, k > 0 ? 1u : 0u);
                        if (!one) {
                            umma_f16_w(d_tmem, ah0 + 16u * k, bl0 + 16u * k, 1u);
                            umma_f16_w(d_tmem, al0 + 16u * k, bh0 + 16u * k, 1u);
                        }
                    }
                    // augmented step: + 2^14 (-|x~|^2 2^-15) = -|x~|^2 / 2
                    if (AUG) umma_f16_w(d_tmem, aug_a, aug_b, 1u);
                }
                }
                umma_commit_w(&bempty[s]);  // operands consumed: the producer may refill stage s
                }
                if (end) break;
                umma_commit_w(&tfull[ts]);  // accumulator ready
                TL(8, it);
            }
#ifdef SLK_WATCHDOG
            ((volatile int *)misc->dbg)[3] = -2;
#endif
        }
        __syncwarp();
    } else if (warp >= 4) {
        // ===================== epilogue warps: one query row per thread
        const int ew = (warp - 4) & 3;   // TMEM lane quarter
        const int grp = (warp - 4) >> 2;  // epilogue group: query block of the group, or column half (HS = 2)
        const int qbi = HS == 2 ? 0 : grp;
        const int half = HS == 2 ? grp : 0;
        const int row = ew * 32 + lane;
        const int64_t gi = (qb + qbi) * BM + row;
        // qid (gathered queries): id of the row in the index, -1 for padding
        const int64_t self_id = (gi < a.nq && a.qid) ? (int64_t)a.qid[gi] : gi;
        const bool row_ok = gi < a.nq && self_id >= 0;
        float qq = 0.0f;  // |q~|^2, written by the convert warps: read after the first tfull
        const int qc = (MODE == MODE_COLOR && row_ok) ? a.qcolor[gi] : -1;
        float *stg = s_stg + (grp * BM + row) * STG_STRIDE;
        // This thread's row keeps its KP best (b, id) pairs in registers,
        // ascending, where b = |x~|^2 - 2<q~,x~> (a = |q~|^2 + b).  thr = the
        // KP-th b; padding rows use -inf so they never take a candidate.  Ties
        // may be ordered either way: the certificate only needs every dropped
        // b >= thr.
        float lv[KP];
        int li[KP];
#pragma unroll
        for (int p = 0; p < KP; p++) {
            lv[p] = INFINITY;
            li[p] = -1;
        }
        float thr = row_ok ? INFINITY : -INFINITY;
#ifdef SLK_TIMELINE
        unsigned long long n_chunk = 0, n_hit = 0, n_iter = 0, n_exam = 0, n_ins = 0;
#endif

        for (int it = 0;; it++) {
            const int ts = it % NT;
            const uint32_t tph = (uint32_t)(it / NT) & 1u;
            if (warp == 4 && lane == 0) TL(9, it);
            mbar_wait(&tfull[ts], tph, 6, it);
            tc_fence_after();
            if (warp == 4 && lane == 0) TL(10, it);
            // the convert warps wrote A (and |q~|^2) before their first bfull arrive
            if (it == 0) qq = s_qq[qbi * BM + row];
            const int slot = it % NMETA;
            const int jb = misc->meta_blk[slot];
#ifdef SLK_WATCHDOG
            if (row == 5) misc->dbg[2] = it * 100000 + (jb < 0 ? 99999 : jb % 100000);
#endif
            if (jb < 0) break;
            const int64_t col0 = (int64_t)jb * BN;
            const uint32_t taddr = tmem + ((uint32_t)(ew * 32) << 16) + (uint32_t)(ts * QB + qbi) * 128;
            // columns this row may take from this block: inside the index, not itself
            const int64_t rem = a.nx - col0;
            const int col_limit = row_ok ? (rem < BN ? (int)rem : BN) : 0;
            const int64_t self_at = a.self_pos ? gi : self_id;
            const int self_col =
                (MODE == MODE_SELF && self_at >= col0 && self_at < col0 + BN) ? (int)(self_at - col0) : -1;
            const int *xcs = s_xcol + slot * BN;
#pragma unroll 1
            for (int c0 = half * (BN / HS); c0 < (half + 1) * (BN / HS); c0 += CH) {
                float dot[CH];
                __syncwarp();  // tcgen05.ld is .sync.aligned: reconverge after the insertion loop
                tmem_ld(taddr + c0, dot);
                // fast path.  AUG: acc = -b / 2, hit iff max(acc) > -thr / 2 (exact
                // scalings).  Else b = fma(-2, acc, |x~|^2) (|x~|^2 from smem), hit
                // iff min(b) < thr.
                float av[CH];
                if (!AUG) {
                    const float *xxs = s_xx + slot * BN;
#pragma unroll
                    for (int i = 0; i < CH; i += 4) {
                        const float4 x4 = *reinterpret_cast<const float4 *>(xxs + c0 + i);
                        av[i + 0] = __fmaf_rn(-2.0f, dot[i + 0], x4.x);
                        av[i + 1] = __fmaf_rn(-2.0f, dot[i + 1], x4.y);
                        av[i + 2] = __fmaf_rn(-2.0f, dot[i + 2], x4.z);
                        av[i + 3] = __fmaf_rn(-2.0f, dot[i + 3], x4.w);
                    }
                }
                float mx[CH / 2];
#pragma unroll
                for (int i = 0; i < CH / 2; i++)
                    mx[i] = AUG ? fmaxf(dot[i], dot[i + CH / 2]) : fminf(av[i], av[i + CH / 2]);
#pragma unroll
                for (int w = CH / 4; w; w >>= 1)
#pragma unroll
                    for (int i = 0; i < w; i++) mx[i] = AUG ? fmaxf(mx[i], mx[i + w]) : fminf(mx[i], mx[i + w]);
                const bool hit = AUG ? mx[0] > -0.5f * thr : mx[0] < thr;
#ifdef SLK_TIMELINE
                n_chunk++;
#endif
                if (!__any_sync(FULL, hit)) continue;  // warp-uniform: nothing to insert
                uint32_t pass = 0;
                if (hit) {
                    // AUG: b = -2 acc exactly, so b < thr <=> acc > -thr / 2; the
                    // chunk is staged as raw accumulators and scaled per insertion
                    const float nthr = -0.5f * thr;
#pragma unroll
                    for (int i = 0; i < CH; i++) pass |= ((AUG ? dot[i] > nthr : av[i] < thr) ? 1u : 0u) << i;
                    uint32_t valid = c0 >= col_limit ? 0u
                                     : (col_limit - c0 >= CH ? CH_ALL : ((1u << (col_limit - c0)) - 1u));
                    if (self_col >= c0 && self_col < c0 + CH) valid &= ~(1u << (self_col - c0));
                    pass &= valid;
                    if (MODE == MODE_COLOR && pass) {
#pragma unroll
                        for (int i = 0; i < CH; i++)
                            if (xcs[c0 + i] == qc) pass &= ~(1u << i);
                    }
                    if (MODE == MODE_SELF && a.xcolor && pass) {
#pragma unroll
                        for (int i = 0; i < CH; i++)
                            if (xcs[c0 + i] < 0) pass &= ~(1u << i);
                    }
                    if (MODE == MODE_MASK && pass) {
                        for (int i = 0; i < CH; i++)
                            if (((pass >> i) & 1u) && a.mask[gi * a.nx + col0 + c0 + i] == 0) pass &= ~(1u << i);
                    }
                    if (pass) {
                        // stage the chunk: a passing value is one LDS away (no
                        // dynamic register indexing)
#pragma unroll
                        for (int i = 0; i < CH; i += 4) {
                            const float *src = AUG ? dot : av;
                            *reinterpret_cast<float4 *>(stg + i) = make_float4(src[i], src[i + 1], src[i + 2], src[i + 3]);
                        }
                    }
                }
#ifdef SLK_TIMELINE
                n_hit++;
                n_iter += __reduce_max_sync(FULL, (unsigned)__popc(pass));
                n_exam += __popc(pass);
#endif
                while (pass) {
                    const int i = __ffs(pass) - 1;
                    pass &= pass - 1;
                    const float v = AUG ? -2.0f * stg[i] : stg[i];
                    if (!(v < thr)) continue;  // the threshold may have dropped
#ifdef SLK_TIMELINE
                    n_ins++;
#endif
                    const int id = (int)(col0 + c0 + i);
                    // shift-insert: new[p] = v < old[p-1] ? old[p-1] : (v < old[p] ? v : old[p])
                    bool c_next = v < lv[KP - 1];
#pragma unroll
                    for (int p = KP - 1; p > 0; p--) {
                        const bool c_prev = v < lv[p - 1];
                        lv[p] = c_prev ? lv[p - 1] : (c_next ? v : lv[p]);
                        li[p] = c_prev ? li[p - 1] : (c_next ? id : li[p]);
                        c_next = c_prev;
                    }
                    if (c_next) {
                        lv[0] = v;
                        li[0] = id;
                    }
                    thr = lv[KP - 1];
                }
            }
            __syncwarp();
            tc_fence_before();
            mbar_arrive(&tempty[ts]);  // accumulator stage free (xx/xcol slots: see NMETA)
            if (warp == 4 && lane == 0) TL(11, it);
            // largest row threshold in a units, rounded up (pruning stays conservative)
            float wm = row_ok ? __fadd_ru(thr, qq) : -INFINITY;
            for (int o = 16; o; o >>= 1) wm = fmaxf(wm, __shfl_xor_sync(FULL, wm, o));
            if (lane == 0) atomicExch(&misc->part[grp * 4 + ew], wm);
        }
#ifdef SLK_TIMELINE
        for (int o = 16; o; o >>= 1) {
            n_exam += __shfl_xor_sync(FULL, n_exam, o);
            n_ins += __shfl_xor_sync(FULL, n_ins, o);
        }
        if (lane == 0) {
            TLC(0, n_chunk);
            TLC(1, n_hit);
            TLC(2, n_iter);
            TLC(3, n_exam);
            TLC(4, n_ins);
        }
#endif
        // write this row's candidate list (slots >= KP hold -1)
        if (gi >= a.row0 && gi < a.row1 && row_ok) {
            const int64_t slot = ((gi - a.row0) * a.nsplit + split) * HS + half;
            int32_t *dst = a.cand + slot * 32;
#pragma unroll
#pragma unroll
            for (int q = 0; q < 32; q++) {
                const int id = q < KP ? li[q < KP ? q : 0] : -1;
                dst[q] = (a.xid && id >= 0) ? a.xid[id] : id;
            }
            // a = |q~|^2 + b rounded down: a lower bound keeps the certificate rigorous
            a.kth[slot] = li[KP - 1] >= 0 ? __fadd_rd(lv[KP - 1], qq) : INFINITY;
            a.qhat[gi - a.row0] = qq;
        }
    }
#ifdef SLK_WATCHDOG
    if (warp != 8) {
        long long w = 0;
        while (++w < (1ll << 24)) {
            if (((volatile int *)misc->dbg)[3] < -1) break;
        }
        if (w >= (1ll << 24) && (tid == 0 || tid == 320 || tid == 128 || tid == 288))
            printf("exit-wait: block %d tid %d dbg %d %d %d %d meta %d %d %d %d %d %d %d %d\n", blockIdx.x, tid,
                   misc->dbg[0], misc->dbg[1], misc->dbg[2], misc->dbg[3], misc->meta_blk[0],
                   misc->meta_blk[1], misc->meta_blk[2], misc->meta_blk[3], misc->meta_blk[4],
                   misc->meta_blk[5], misc->meta_blk[6], misc->meta_blk[7]);
    }
#endif
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == Cfg<EW>::WARP_MMA) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS)
                     : "memory");
    }
}

template <int MODE, int KP, bool AUG, int QB, bool CK, int HS = 1>
void launch_mode(const TcArgs &args, int64_t ngroups, cudaStream_t s) {
    const Plan P = make_plan(args.dk, AUG, QB, CK ? KC : 0, QB * HS);
    SLK_CUDA(cudaFuncSetAttribute(tc_scan_kernel<MODE, KP, AUG, QB, CK, HS>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P.total));
    tc_scan_kernel<MODE, KP, AUG, QB, CK, HS>
        <<<(unsigned)(ngroups * args.nsplit), Cfg<QB * HS>::NTHREADS, P.total, s>>>(args);
    SLK_CHECK_LAUNCH();
}

template <int KP, bool AUG, int QB, bool CK = false>
void launch_kp(int mode, const TcArgs &args, int64_t ngroups, cudaStream_t s) {
    switch (mode) {
        case MODE_NONE: launch_mode<MODE_NONE, KP, AUG, QB, CK>(args, ngroups, s); break;
        case MODE_MASK: launch_mode<MODE_MASK, KP, AUG, QB, CK>(args, ngroups, s); break;
        case MODE_COLOR: launch_mode<MODE_COLOR, KP, AUG, QB, CK>(args, ngroups, s); break;
        default: launch_mode<MODE_SELF, KP, AUG, QB, CK>(args, ngroups, s); break;
    }
}

void launch_ck(int mode, int kp, const TcArgs &args, int64_t ngroups, cudaStream_t s) {
    if (kp <= 2) launch_kp<2, false, 1, true>(mode, args, ngroups, s);
    else if (kp <= 4) launch_kp<4, false, 1, true>(mode, args, ngroups, s);
    else if (kp <= 8) launch_kp<8, false, 1, true>(mode, args, ngroups, s);
    else if (kp <= 16) launch_kp<16, false, 1, true>(mode, args, ngroups, s);
    else launch_kp<32, false, 1, true>(mode, args, ngroups, s);
}

// the k-NN pass with column halves (HS = 2)
template <bool AUG>
void launch_halves_t(int mode, int kp, const TcArgs &args, int64_t ngroups, cudaStream_t s) {
    if (mode == MODE_COLOR) launch_mode<MODE_COLOR, 8, AUG, 1, false, 2>(args, ngroups, s);
    else if (kp <= 8) launch_mode<MODE_SELF, 8, AUG, 1, false, 2>(args, ngroups, s);
    else launch_mode<MODE_SELF, 16, AUG, 1, false, 2>(args, ngroups, s);
}

template <bool AUG>
void launch_aug(int mode, int kp, int qb, const TcArgs &args, int64_t ngroups, cudaStream_t s) {
    if (qb == 2) {
        if (kp <= 2) launch_kp<2, AUG, 2>(mode, args, ngroups, s);
        else if (kp <= 4) launch_kp<4, AUG, 2>(mode, args, ngroups, s);
        else if (kp <= 8) launch_kp<8, AUG, 2>(mode, args, ngroups, s);
        else launch_kp<16, AUG, 2>(mode, args, ngroups, s);
        return;
    }
    if (kp <= 2) launch_kp<2, AUG, 1>(mode, args, ngroups, s);
    else if (kp <= 4) launch_kp<4, AUG, 1>(mode, args, ngroups, s);
    else if (kp <= 8) launch_kp<8, AUG, 1>(mode, args, ngroups, s);
    else if (kp <= 16) launch_kp<16, AUG, 1>(mode, args, ngroups, s);
    else launch_kp<32, AUG, 1>(mode, args, ngroups, s);
}

}  // namespace

void timeline_arm(cudaStream_t s) { tl_arm(s); }
void timeline_dump(int mode, int64_t rows, cudaStream_t s) { tl_dump(mode, rows, s); }

int nprod_for(bool rerun) {
    if (const char *e = getenv("SLK_TC_NPROD")) {
        const int v = atoi(e);
        if (v == 1 || v == 3) return v;
    }
    (void)rerun;
    // measured at C3 (round 2): one product leaves 5 % of the cross-colour rows
    // uncertified and its K' = 32 reruns cost more than the scan saves
    return 3;
}

static int round16(int d) { return ((d + 15) / 16) * 16; }
static bool aug_fits(int d) { return make_plan(round16(d), true, 1).nb >= 3; }

// Chunked (large-d) kernel when the whole-block kernel cannot hold its A
// tile plus two B stages (d > 128)
bool chunked(int d) { return make_plan(round16(d), aug_fits(d), 1).nb < 2; }

// The augmented norm step when at least 3 B stages still fit (measured: the
// max-only epilogue pays for the extra MMA and the 16 extra K columns);
// otherwise |x~|^2 goes through shared memory (large d).
bool use_aug(int d) { return !chunked(d) && aug_fits(d); }

// chunked: whole 64-dim TMEM stores of the query's hi term
int k_extent(int d) { return chunked(d) ? ((d + 63) / 64) * 64 : round16(d); }

int chunk_dims(int d) { return chunked(d) ? KC : k_extent(d); }

size_t smem_bytes(int d) {
    return chunked(d) ? make_plan(k_extent(d), false, 1, KC).total : make_plan(k_extent(d), use_aug(d), 1).total;
}

// at least two B stages must fit next to the A tile; chunked: the query's hi
// term must fit in TMEM next to two accumulator stages
bool supported(int d) {
    if (!chunked(d)) return true;
    return k_extent(d) <= CK_MAX_DK && make_plan(k_extent(d), false, 1, KC).nb >= 2;
}

// query blocks per CTA for K' = kp candidates: pairs need K' <= 16 (the 8
// epilogue warps cap registers) and 2 B stages next to two A tiles
// Measured: pairs cut the cross-colour passes by 13 % at C3 (blocks of one
// cluster pair well) but the union of two blocks' visit lists costs 1.4-2.5x
// the tiles when clusters span only a few blocks (C5): knn.cu:tc_pass uses
// them only when the pair spheres are nearly as tight as the blocks'
// (SLK_TC_QB=1 / 2 force singles / pairs).
int group_blocks(int d, int kp) {
    const char *e = getenv("SLK_TC_QB");
    if ((e && atoi(e) == 1) || kp > 16 || chunked(d)) return 1;
    return make_plan(k_extent(d), use_aug(d), 2).nb >= 2 ? 2 : 1;
}

// k-NN pass (MODE_SELF) with two column-half lists per row: K' <= 16, the
// whole-block kernel, and the extra epilogue staging must still leave two B
// stages (three with the augmented step)
bool halves_supported(int mode, int d, int kp) {
    if (chunked(d) || kp > 16 || (mode != MODE_SELF && mode != MODE_COLOR) || (mode == MODE_COLOR && kp > 8))
        return false;
    // k-NN lists of K' = 8 (k < 8): one list per row is faster than two of 8
    // (C5, k = 2: scan 8.2 -> 7.4 ms, refine 1.0 -> 0.6 ms); the halves pay
    // off for K' = 16 (C3: scan 19.4 -> 17.6 ms)
    if (mode == MODE_SELF && kp < 16) return false;
    if (const char *e = getenv("SLK_TC_HS"))
        if (atoi(e) == 1) return false;
    return make_plan(k_extent(d), use_aug(d), 1, 0, 2).nb >= (use_aug(d) ? 3 : 2);
}

void launch_halves(int mode, int kp, const TcArgs &args, int64_t ngroups, cudaStream_t s) {
    if (use_aug(args.d)) launch_halves_t<true>(mode, kp, args, ngroups, s);
    else launch_halves_t<false>(mode, kp, args, ngroups, s);
}

// K' = kp candidates per row (2, 4, 8, 16 or 32; kp > k for the certificate);
// qb query blocks per CTA (group_blocks), ngroups groups in the launch
void launch(int mode, int kp, int qb, const TcArgs &args, int64_t ngroups, cudaStream_t s) {
    if (chunked(args.d)) launch_ck(mode, kp, args, ngroups, s);
    else if (use_aug(args.d)) launch_aug<true>(mode, kp, qb, args, ngroups, s);
    else launch_aug<false>(mode, kp, qb, args, ngroups, s);
}

}  // namespace tc
}  // namespace slk
