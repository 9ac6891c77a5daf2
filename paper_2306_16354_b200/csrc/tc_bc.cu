// tc_bc.cu — block-centred one-product tcgen05 scan, sm_100a.
//
// Same contract as tc_scan.cu (the reference's _knn_scan_tile /
// _nn1_scan_tile, /root/reference/pkg/src/parlink/neighbors.py:119-160,
// 191-217): one CTA owns 128 query rows for the whole pruned index sweep and
// leaves, per row, two K'-candidate lists (column halves) by an approximate
// distance; the float64 refine + certificate (knn.cu) makes the result exact.
//
// What differs from tc_scan.cu is where the centring happens:
//
//   * the INDEX is converted once per call (bcpack_kernel): every point is
//     centred on its own block's centroid c_b, scaled by the power of two s and
//     rounded to fp16, x~ = fp16((x - c_b) s), in the canonical K-major
//     no-swizzle UMMA layout, followed by the block's augmented norm tile
//     (-|x~|^2 2^-15 as a two-term fp16 split), -c_b s and the block radius.
//     A tile is one bulk copy of 128 * DK * 2 + 4 KB + ... bytes (20.3 KB at
//     d = 64 against 32 KB of raw fp32) and needs no conversion;
//   * the QUERY rows are re-centred per tile on the visited block's centroid,
//     a = fp16(q s - c_b s), from registers (each convert thread holds its row)
//     straight into tensor memory (tcgen05.st), double-buffered, and the MMA
//     reads A from TMEM (.kind::f16 [d], [a_tmem], b_desc): shared memory only
//     serves B, so an M = 128, N = 128, K = 16 step reads 4 KB instead of 8;
//   * one fp16 product per 16 dims (hi.hi).  The error of <a, x~> is
//     2^-9 |a||x~| with |x~| <= the block radius rho_b: the certificate
//     (knn.cu:certified_floor_bc) uses the largest radius the CTA visited.
//
// CTA = 18 warps (14 at DK = 16), warp-specialised, mbarrier hand-offs:
//   warps 0-3, 14-17    convert: two threads per query row (one per half of the
//                        dims) hold it in registers; per tile a -> TMEM (three
//                        slots, two at DK = 128), |a|^2 halves -> smem ring
//   warps 4-11          epilogue: tcgen05.ld one accumulator row per thread, two
//                        warps per TMEM lane quarter (column halves), fast
//                        max filter, exact pass mask, K'-list insertion
//   warp 12             MMA issue (elect.sync)
//   warp 13             producer: pruned visit order, one bulk copy per block
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

constexpr int NT = 3;                // TMEM accumulator stages (128 columns each)
constexpr int MAX_NB = 8;            // B stages
constexpr int NMETA = MAX_NB + NT + 2;  // per-tile ring: producer runs <= NB + NT tiles ahead of the epilogue
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t ACOL = NT * 128;  // A slots: NA x DK/2 columns after the accumulators
constexpr int NA_MAX = 3;
constexpr int CH = 32;
constexpr int STG_STRIDE = CH + 4;
constexpr uint32_t AUG_TILE = BM * 16 * 2;
constexpr float NORM_A = 16384.0f;        // 2^14
constexpr float NORM_B_SCALE = -0x1p-15f;
constexpr uint32_t SMEM_LIMIT = 227 * 1024;
constexpr int WARP_EPI = 4, WARP_MMA = 12, WARP_PROD = 13, WARP_CONV2 = 14;

// per-block record of the bc-packed index
__host__ __device__ constexpr uint32_t rec_hi(int dk) { return (uint32_t)BM * dk * 2; }
__host__ __device__ constexpr uint32_t rec_cneg(int dk) { return rec_hi(dk) + AUG_TILE; }
__host__ __device__ constexpr uint32_t rec_rho(int dk) { return rec_cneg(dk) + (uint32_t)dk * 4; }
__host__ __device__ constexpr uint32_t rec_bytes(int dk) { return rec_rho(dk) + 16; }
__host__ __device__ constexpr uint32_t stage_stride(int dk) { return (rec_bytes(dk) + 1023) / 1024 * 1024; }

struct Plan {
    uint32_t aaug, xcol, aa, stg, misc, bars, b, total;
    int nb;
};
__host__ __device__ inline Plan make_plan(int dk, int ncg) {
    Plan p{};
    uint32_t off = 0;
    auto take = [&](uint32_t bytes, uint32_t align) {
        off = (off + align - 1) / align * align;
        const uint32_t at = off;
        off += bytes;
        return at;
    };
    p.aaug = take(AUG_TILE, 1024);
    p.xcol = take(NMETA * BN * 4, 16);
    p.aa = take(NMETA * ncg * BM * 4, 16);
    p.stg = take(2 * BM * STG_STRIDE * 4, 16);
    p.misc = take(256, 16);
    p.bars = take(8 * (2 * MAX_NB + 2 * NA_MAX + 2 * NT), 8);
    off = (off + 1023) / 1024 * 1024;
    const uint32_t st = stage_stride(dk);
    const int nb = off >= SMEM_LIMIT ? 0 : (int)((SMEM_LIMIT - off) / st);
    p.nb = nb > MAX_NB ? MAX_NB : nb;
    p.b = take(st * (p.nb > 0 ? p.nb : 0), 1024);
    p.total = off;
    return p;
}

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
    float part[8];       // per epilogue warp: largest row threshold (a units); 16-byte aligned
    uint32_t tmem_base;
    unsigned rho_bits;   // largest block radius visited (scaled, float bits; radii >= 0)
    int meta_blk[NMETA];
};

#ifdef SLK_WATCHDOG
__device__ void watchdog_dump(int tag, int it, uint32_t parity, unsigned long long st) {
    printf("watchdog(bc): block %d thread %d tag %d it %d parity %u state %llx\n", blockIdx.x, threadIdx.x, tag,
           it, parity, st);
}
#endif

template <int N>
__device__ __forceinline__ void tmem_st(uint32_t taddr, const uint32_t (&r)[N]);
template <>
__device__ __forceinline__ void tmem_st<8>(uint32_t taddr, const uint32_t (&r)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
                 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}
template <>
__device__ __forceinline__ void tmem_st<16>(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}
template <>
__device__ __forceinline__ void tmem_st<32>(uint32_t taddr, const uint32_t (&r)[32]) {
    tmem_st32(taddr, r);
}

// Two 32-column accumulator loads, one wait: the wait names every destination
// register as read-write so the compiler keeps all uses after it.
__device__ __forceinline__ void tmem_ld32x2(uint32_t taddr, float (&va)[32], float (&vb)[32]) {
    uint32_t a[32], b[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]), "=r"(a[6]), "=r"(a[7]), "=r"(a[8]), "=r"(a[9]), "=r"(a[10]), "=r"(a[11]), "=r"(a[12]), "=r"(a[13]), "=r"(a[14]), "=r"(a[15]), "=r"(a[16]), "=r"(a[17]), "=r"(a[18]), "=r"(a[19]), "=r"(a[20]), "=r"(a[21]), "=r"(a[22]), "=r"(a[23]), "=r"(a[24]), "=r"(a[25]), "=r"(a[26]), "=r"(a[27]), "=r"(a[28]), "=r"(a[29]), "=r"(a[30]), "=r"(a[31])
        : "r"(taddr));
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(b[0]), "=r"(b[1]), "=r"(b[2]), "=r"(b[3]), "=r"(b[4]), "=r"(b[5]), "=r"(b[6]), "=r"(b[7]), "=r"(b[8]), "=r"(b[9]), "=r"(b[10]), "=r"(b[11]), "=r"(b[12]), "=r"(b[13]), "=r"(b[14]), "=r"(b[15]), "=r"(b[16]), "=r"(b[17]), "=r"(b[18]), "=r"(b[19]), "=r"(b[20]), "=r"(b[21]), "=r"(b[22]), "=r"(b[23]), "=r"(b[24]), "=r"(b[25]), "=r"(b[26]), "=r"(b[27]), "=r"(b[28]), "=r"(b[29]), "=r"(b[30]), "=r"(b[31])
        : "r"(taddr + 32u));
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3]), "+r"(a[4]), "+r"(a[5]), "+r"(a[6]), "+r"(a[7]), "+r"(a[8]), "+r"(a[9]), "+r"(a[10]), "+r"(a[11]), "+r"(a[12]), "+r"(a[13]), "+r"(a[14]), "+r"(a[15]), "+r"(a[16]), "+r"(a[17]), "+r"(a[18]), "+r"(a[19]), "+r"(a[20]), "+r"(a[21]), "+r"(a[22]), "+r"(a[23]), "+r"(a[24]), "+r"(a[25]), "+r"(a[26]), "+r"(a[27]), "+r"(a[28]), "+r"(a[29]), "+r"(a[30]), "+r"(a[31]), "+r"(b[0]), "+r"(b[1]), "+r"(b[2]), "+r"(b[3]), "+r"(b[4]), "+r"(b[5]), "+r"(b[6]), "+r"(b[7]), "+r"(b[8]), "+r"(b[9]), "+r"(b[10]), "+r"(b[11]), "+r"(b[12]), "+r"(b[13]), "+r"(b[14]), "+r"(b[15]), "+r"(b[16]), "+r"(b[17]), "+r"(b[18]), "+r"(b[19]), "+r"(b[20]), "+r"(b[21]), "+r"(b[22]), "+r"(b[23]), "+r"(b[24]), "+r"(b[25]), "+r"(b[26]), "+r"(b[27]), "+r"(b[28]), "+r"(b[29]), "+r"(b[30]), "+r"(b[31])
                 :
                 : "memory");
#pragma unroll
    for (int i = 0; i < 32; i++) {
        va[i] = __uint_as_float(a[i]);
        vb[i] = __uint_as_float(b[i]);
    }
}

// -|x~|^2 2^-15 as hi + lo fp16 (|hi + lo - v| <= 2^-22 |v| + 2^-25)
__device__ __forceinline__ void norm_split(float xx, float &t0, float &t1) {
    const float v = xx * NORM_B_SCALE;  // exact: power of two
    const float hi = __half2float(__float2half_rn(v));
    t0 = hi;
    t1 = __fsub_rn(v, hi);
}

// Index conversion, one CTA of 128 threads per block, one thread per point.
__global__ void __launch_bounds__(128) bcpack_kernel(const float *__restrict__ x, const int32_t *__restrict__ rowmap,
                                                     int64_t n, int d, int dk, int64_t nb,
                                                     const float *__restrict__ centroid,
                                                     const float *__restrict__ radius, float scale,
                                                     unsigned char *__restrict__ out) {
    const int64_t b = blockIdx.x;
    const int r = threadIdx.x;
    const int64_t p = b * BM + r;
    unsigned char *rec = out + b * (int64_t)rec_bytes(dk);
    float *cneg = reinterpret_cast<float *>(rec + rec_cneg(dk));
    for (int t = r; t < dk; t += BM) cneg[t] = t < d ? -centroid[(int64_t)t * nb + b] * scale : 0.0f;
    if (r == 0) {
        float *rho = reinterpret_cast<float *>(rec + rec_rho(dk));
        // |fl(x s - c s)| <= rho s (1 + 2^-24); the radius already carries 1e-6
        rho[0] = radius[b] * scale;
        rho[1] = rho[2] = rho[3] = 0.0f;
    }
    __syncthreads();
    const bool real = p < n;
    const float *xr = x + (real ? (rowmap ? (int64_t)rowmap[p] : p) : 0) * d;
    unsigned char *row = rec + (r >> 3) * (dk * 16) + (r & 7) * 16;
    float nrm4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    for (int g = 0; g < dk / 8; g++) {
        __half2 h[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {
            float v[2];
#pragma unroll
            for (int e = 0; e < 2; e++) {
                const int t = 8 * g + 2 * q + e;
                v[e] = (real && t < d) ? __fmaf_rn(xr[t], scale, cneg[t]) : 0.0f;
                nrm4[q] = __fmaf_rn(v[e], v[e], nrm4[q]);
            }
            h[q] = __floats2half2_rn(v[0], v[1]);
        }
        *reinterpret_cast<uint4 *>(row + g * 128) = *reinterpret_cast<uint4 *>(h);
    }
    const float xx = __fadd_rn(__fadd_rn(nrm4[0], nrm4[1]), __fadd_rn(nrm4[2], nrm4[3]));
    float t0, t1;
    norm_split(xx, t0, t1);
    unsigned char *aug = rec + rec_hi(dk) + (r >> 3) * 256 + (r & 7) * 16;
    const __half2 h0 = __floats2half2_rn(t0, t1), z = __floats2half2_rn(0.0f, 0.0f);
    *reinterpret_cast<uint4 *>(aug) =
        make_uint4(*reinterpret_cast<const uint32_t *>(&h0), *reinterpret_cast<const uint32_t *>(&z),
                   *reinterpret_cast<const uint32_t *>(&z), *reinterpret_cast<const uint32_t *>(&z));
    *reinterpret_cast<uint4 *>(aug + 128) = make_uint4(0u, 0u, 0u, 0u);
}

// One convert thread per row, two (one per half of the dims) when the row
// would not fit one thread's registers (DK = 128).  The register file is
// split over the four SM sub-partitions: 14 warps allow 128 registers per
// thread, 18 warps 96.
#ifndef SLK_BC_NCG2_MIN_DK
#define SLK_BC_NCG2_MIN_DK 128
#endif
template <int DK, int KP>
struct Shape {
    static constexpr int NCG = DK >= SLK_BC_NCG2_MIN_DK ? 2 : 1;  // convert warp groups
    static constexpr int DC = DK / NCG;           // dims per convert thread
    static constexpr int NTHREADS = (14 + 4 * (NCG - 1)) * 32;
    static constexpr int NA = DK <= 64 ? 3 : 2;   // A slots in TMEM (NT * 128 + NA * DK / 2 <= 512)
};

template <int MODE, int KP, int DK>
__global__ void __launch_bounds__(Shape<DK, KP>::NTHREADS, 1) tc_bc_kernel(TcArgs a) {
    extern __shared__ __align__(1024) unsigned char smem[];
    constexpr int NCG = Shape<DK, KP>::NCG, DC = Shape<DK, KP>::DC, NA = Shape<DK, KP>::NA;
    constexpr uint32_t REC = rec_bytes(DK), STAGE = stage_stride(DK);
    const Plan P = make_plan(DK, NCG);
    const int nb = P.nb;
    unsigned char *sB = smem + P.b;
    unsigned char *sAaug = smem + P.aaug;
    int *s_xcol = reinterpret_cast<int *>(smem + P.xcol);
    float *s_aa = reinterpret_cast<float *>(smem + P.aa);
    float *s_stg = reinterpret_cast<float *>(smem + P.stg);
    Misc *misc = reinterpret_cast<Misc *>(smem + P.misc);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + P.bars);  // producer (bulk copy) -> MMA / convert
    uint64_t *empty = full + MAX_NB;                                // MMA commit -> producer
    uint64_t *afull = empty + MAX_NB;                               // convert -> MMA (A slot written)
    uint64_t *aempty = afull + NA_MAX;                              // MMA commit -> convert
    uint64_t *tfull = aempty + NA_MAX;                              // MMA commit -> epilogue
    uint64_t *tempty = tfull + NT;                                  // epilogue -> MMA

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t qbl = blockIdx.x / a.nsplit;
    const int split = blockIdx.x - (int)qbl * a.nsplit;
    const int64_t qb = a.qb0 + qbl;

    if (tid == 0) {
        for (int s = 0; s < MAX_NB; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < NA; s++) {
            mbar_init(&afull[s], 128 * NCG);
            mbar_init(&aempty[s], 1);
        }
        for (int s = 0; s < NT; s++) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], 256);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int i = 0; i < 8; i++) misc->part[i] = INFINITY;
        misc->rho_bits = 0u;
    }
    if (warp == WARP_MMA) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&misc->tmem_base)),
                     "r"(TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    // augmented-step A tile: columns 0, 1 = 2^14, the rest zero.  Canonical
    // layout: 16-byte segment e holds row (e >> 4) * 8 + (e & 7), K half
    // (e >> 3) & 1; columns 0, 1 are the first 4 bytes of the K-half-0 segments
    for (uint32_t e = tid; e < AUG_TILE / 16; e += blockDim.x) {
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (((e >> 3) & 1u) == 0u) {
            const __half2 h = __floats2half2_rn(NORM_A, NORM_A);
            v.x = *reinterpret_cast<const uint32_t *>(&h);
        }
        reinterpret_cast<uint4 *>(sAaug)[e] = v;
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = misc->tmem_base;

    if (warp == WARP_PROD) {
        // ===================== producer: visit order + one bulk copy per block
        BlockVisitor vis(a.sb_order + qbl * a.nsb, a.sb_lb + qbl * a.nsb, a.flat_lb + qbl * a.nsb * 32,
                         a.nvalid[qbl], lane, split, a.nsplit);
        int64_t computed = 0;
        Ring rg{0, 0u, nb};
        const bool col = MODE == MODE_COLOR || (MODE == MODE_SELF && a.xcolor);
        for (int it = 0;; it++, rg.next()) {
            // the epilogue warps publish their largest row threshold with an
            // atomic exchange; two volatile 16-byte reads see each slot whole,
            // and thresholds only shrink, so any value read is a valid bound
            float thr;
            {
                float4 p0, p1;
                const uint32_t pa = smem_u32(misc->part);
                asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                             : "=f"(p0.x), "=f"(p0.y), "=f"(p0.z), "=f"(p0.w) : "r"(pa));
                asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                             : "=f"(p1.x), "=f"(p1.y), "=f"(p1.z), "=f"(p1.w) : "r"(pa + 16));
                thr = fmaxf(fmaxf(fmaxf(p0.x, p0.y), fmaxf(p0.z, p0.w)), fmaxf(fmaxf(p1.x, p1.y), fmaxf(p1.z, p1.w)));
                thr *= a.inv_scale2;
            }
            if (lane == 0) TL(12, it);
            const int64_t jb = vis.next(thr, lane);
            if (lane == 0) {
                TL(0, it);
                mbar_wait(&empty[rg.s], rg.ph ^ 1u, 1, it);
                TL(1, it);
                misc->meta_blk[it % NMETA] = (int)jb;
                if (jb < 0) {
                    mbar_arrive(&full[rg.s]);
                } else {
                    mbar_expect_tx(&full[rg.s], REC + (col ? BN * 4 : 0));
                    bulk_g2s(sB + (size_t)rg.s * STAGE, a.bcx + jb * (int64_t)REC, REC, &full[rg.s]);
                    if (col) bulk_g2s(s_xcol + (it % NMETA) * BN, a.xcolor + jb * BN, BN * 4, &full[rg.s]);
                    computed++;
                }
                TL(2, it);
            }
            if (jb < 0) break;
        }
        if (lane == 0 && a.tiles_done) atomicAdd(a.tiles_done, (unsigned long long)computed);
    } else if (warp < 4 || (NCG == 2 && warp >= WARP_CONV2)) {
        // ===================== convert: a = fp16(q s - c_b s) of this row -> TMEM
        const int g = warp < 4 ? 0 : 1;           // dims [g DC, g DC + DC)
        const int r = (warp & 3) * 32 + lane;     // TMEM lane quarter = warp % 4
        const int64_t gi = qb * BM + r;
        float q[DC];
        {
            const bool ok = gi < a.nq;
            const float *qr = a.qp + (ok ? gi : 0) * (int64_t)a.d;
#pragma unroll
            for (int t = 0; t < DC; t++) {
                const int tt = g * DC + t;
                q[t] = (ok && tt < a.d) ? qr[tt] * a.scale : 0.0f;  // exact: power of two
            }
        }
        const uint32_t lane_base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + ACOL + (uint32_t)g * (DC / 2);
        Ring rg{0, 0u, nb};
        for (int it = 0;; it++, rg.next()) {
            mbar_wait(&full[rg.s], rg.ph, 3, it);
            if (r == 0 && g == 0) TL(3, it);
            const int jb = misc->meta_blk[it % NMETA];
            if (jb < 0) break;
            const int slot = it % NA;
            mbar_wait(&aempty[slot], ((uint32_t)(it / NA) & 1u) ^ 1u, 7, it);
            const unsigned char *rec = sB + (size_t)rg.s * STAGE;
            const float *cneg = reinterpret_cast<const float *>(rec + rec_cneg(DK)) + g * DC;
            uint32_t h[DC / 2];
            float n4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#ifdef SLK_ABL_NOCONV
            if (false)
#endif
#pragma unroll
            for (int t = 0; t < DC; t += 4) {
                const float4 c = *reinterpret_cast<const float4 *>(cneg + t);
                const float v0 = __fadd_rn(q[t], c.x), v1 = __fadd_rn(q[t + 1], c.y);
                const float v2 = __fadd_rn(q[t + 2], c.z), v3 = __fadd_rn(q[t + 3], c.w);
                n4[0] = __fmaf_rn(v0, v0, n4[0]);
                n4[1] = __fmaf_rn(v1, v1, n4[1]);
                n4[2] = __fmaf_rn(v2, v2, n4[2]);
                n4[3] = __fmaf_rn(v3, v3, n4[3]);
                const __half2 h01 = __floats2half2_rn(v0, v1), h23 = __floats2half2_rn(v2, v3);
                h[t / 2] = *reinterpret_cast<const uint32_t *>(&h01);
                h[t / 2 + 1] = *reinterpret_cast<const uint32_t *>(&h23);
            }
            tmem_st<DC / 2>(lane_base + (uint32_t)slot * (DK / 2), h);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            s_aa[((it % NMETA) * NCG + g) * BM + r] = __fadd_rn(__fadd_rn(n4[0], n4[1]), __fadd_rn(n4[2], n4[3]));
            if (r == 0 && g == 0)
                atomicMax(&misc->rho_bits, __float_as_uint(*reinterpret_cast<const float *>(rec + rec_rho(DK))));
            tc_fence_before();
            mbar_arrive(&afull[slot]);  // every thread arrives: its writes are released by its own arrive
            if (r == 0 && g == 0) TL(4, it);
        }
    } else if (warp == WARP_MMA) {
        // ===================== MMA issuer (whole warp; elect.sync issues)
        const uint32_t b_base = smem_u32(sB);
        const uint64_t aug_a = umma_desc(smem_u32(sAaug), 128, 256);
        constexpr uint32_t SBO = (uint32_t)DK * 16;
        Ring rg{0, 0u, nb};
        for (int it = 0;; it++, rg.next()) {
            const int ts = it % NT;
            const uint32_t tph = (uint32_t)(it / NT) & 1u;
            TL(5, it);
            mbar_wait(&full[rg.s], rg.ph, 4, it);
            TL(6, it);
            mbar_wait(&tempty[ts], tph ^ 1u, 5, it);
            if (misc->meta_blk[it % NMETA] < 0) {
                if (lane == 0) mbar_arrive(&tfull[ts]);
                break;
            }
            const int slot = it % NA;
            mbar_wait(&afull[slot], (uint32_t)(it / NA) & 1u, 8, it);
            TL(7, it);
            tc_fence_after();
            const uint32_t bs = b_base + rg.s * STAGE;
            const uint32_t d_tmem = tmem + (uint32_t)ts * 128;
            const uint32_t a_tmem = tmem + ACOL + (uint32_t)slot * (DK / 2);
            const uint64_t b0 = umma_desc(bs, 128, SBO);
#ifndef SLK_ABL_NOMMA
#pragma unroll
            for (int k = 0; k < DK / 16; k++) umma_f16_ta_w(d_tmem, a_tmem + 8u * k, b0 + 16u * k, k > 0 ? 1u : 0u);
            // augmented step: + 2^14 (-|x~|^2 2^-15) = -|x~|^2 / 2
            umma_f16_w(d_tmem, aug_a, umma_desc(bs + rec_hi(DK), 128, 256), 1u);
#else
            (void)a_tmem;
            (void)b0;
            (void)aug_a;
#endif
            umma_commit_w(&empty[rg.s]);
            umma_commit_w(&aempty[slot]);
            umma_commit_w(&tfull[ts]);
            TL(8, it);
        }
        __syncwarp();
    } else if (warp >= WARP_EPI && warp < WARP_MMA) {
        // ===================== epilogue: one query row per thread, column halves
        const int ew = warp & 3;             // TMEM lane quarter
        const int half = (warp - WARP_EPI) >> 2;
        const int row = ew * 32 + lane;
        const int64_t gi = qb * BM + row;
        const int64_t self_id = (gi < a.nq && a.qid) ? (int64_t)a.qid[gi] : gi;
        const bool row_ok = gi < a.nq && self_id >= 0;
        const int qc = (MODE == MODE_COLOR && row_ok) ? a.qcolor[gi] : -1;
        float *stg = s_stg + (half * BM + row) * STG_STRIDE;
        // K' best (v, id), ascending, v = |a|^2 - 2 acc rounded down (a lower
        // bound of the exact value of the computed terms); thr = the K'-th.
        float lv[KP];
        int li[KP];
#pragma unroll
        for (int p = 0; p < KP; p++) {
            lv[p] = INFINITY;
            li[p] = -1;
        }
        float thr = row_ok ? INFINITY : -INFINITY;
        for (int it = 0;; it++) {
            const int ts = it % NT;
            const uint32_t tph = (uint32_t)(it / NT) & 1u;
            if (warp == WARP_EPI && lane == 0) TL(9, it);
#ifdef SLK_EPI_SPIN
            mbar_wait_spin(&tfull[ts], tph);
#else
            mbar_wait(&tfull[ts], tph, 6, it);
#endif
            tc_fence_after();
            if (warp == WARP_EPI && lane == 0) TL(10, it);
            const int slot = it % NMETA;
            const int jb = misc->meta_blk[slot];
            if (jb < 0) break;
            float aa = s_aa[(slot * NCG) * BM + row];
            if (NCG == 2) aa = __fadd_rn(aa, s_aa[(slot * NCG + 1) * BM + row]);
            const int64_t col0 = (int64_t)jb * BN;
            const uint32_t taddr = tmem + ((uint32_t)(ew * 32) << 16) + (uint32_t)ts * 128;
            const int64_t rem = a.nx - col0;
            const int col_limit = row_ok ? (rem < BN ? (int)rem : BN) : 0;
            const int64_t self_at = a.self_pos ? gi : (a.xpos && self_id >= 0 ? (int64_t)a.xpos[self_id] : self_id);
            const int self_col =
                (MODE == MODE_SELF && self_at >= col0 && self_at < col0 + BN) ? (int)(self_at - col0) : -1;
            const int *xcs = s_xcol + slot * BN;
            // acc > nthr <=> |a|^2 - 2 acc < thr; nthr rounded down, so every
            // dropped column has exact |a|^2 - 2 acc >= thr
            float nthr = 0.5f * __fsub_rd(aa, thr);
            // one 32-column chunk: fast max filter, exact pass mask, insertion
            auto chunk = [&](const float (&dot)[CH], const int c0) {
                float mx[CH / 2];
#pragma unroll
                for (int i = 0; i < CH / 2; i++) mx[i] = fmaxf(dot[i], dot[i + CH / 2]);
#pragma unroll
                for (int w = CH / 4; w; w >>= 1)
#pragma unroll
                    for (int i = 0; i < w; i++) mx[i] = fmaxf(mx[i], mx[i + w]);
                const bool hit = mx[0] > nthr;
                if (!__any_sync(FULL, hit)) return;
                uint32_t pass = 0;
                if (hit) {
#pragma unroll
                    for (int i = 0; i < CH; i++) pass |= (dot[i] > nthr ? 1u : 0u) << i;
                    uint32_t valid = c0 >= col_limit ? 0u
                                     : (col_limit - c0 >= CH ? 0xffffffffu : ((1u << (col_limit - c0)) - 1u));
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
                    if (pass) {
#pragma unroll
                        for (int i = 0; i < CH; i += 4)
                            *reinterpret_cast<float4 *>(stg + i) = make_float4(dot[i], dot[i + 1], dot[i + 2], dot[i + 3]);
                    }
                }
                while (pass) {
                    const int i = __ffs(pass) - 1;
                    pass &= pass - 1;
                    const float v = __fmaf_rd(-2.0f, stg[i], aa);
                    if (!(v < thr)) continue;
                    const int id = (int)(col0 + c0 + i);
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
                nthr = 0.5f * __fsub_rd(aa, thr);
            };
#ifdef SLK_ABL_NOEPI
            if (false)
#endif
            if (KP <= 8) {
                // K' = 8: both chunks of the half in one TMEM round trip
                float da[CH], db[CH];
                __syncwarp();
                tmem_ld32x2(taddr + half * 64, da, db);
                chunk(da, half * 64);
                chunk(db, half * 64 + CH);
            } else {
#pragma unroll 1
                for (int c0 = half * 64; c0 < half * 64 + 64; c0 += CH) {
                    float dot[CH];
                    __syncwarp();
                    tmem_ld32(taddr + c0, dot);
                    chunk(dot, c0);
                }
            }
            __syncwarp();
            tc_fence_before();
            mbar_arrive(&tempty[ts]);
            if (warp == WARP_EPI && lane == 0) TL(11, it);
            // warp maximum of the row thresholds in one REDUX (order-preserving
            // float -> uint map), published for the producer's pruning
#ifdef SLK_PUB2
            if (it & 1)
#endif
            {
                const uint32_t b = __float_as_uint(row_ok ? thr : -INFINITY);
                const uint32_t key = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
                const uint32_t mk = __reduce_max_sync(FULL, key);
                const uint32_t mb = (mk & 0x80000000u) ? (mk & 0x7fffffffu) : ~mk;
                if (lane == 0) atomicExch(&misc->part[warp - WARP_EPI], __uint_as_float(mb));
            }
        }
        if (gi >= a.row0 && gi < a.row1 && row_ok) {
            const int64_t slot = ((gi - a.row0) * a.nsplit + split) * 2 + half;
            int32_t *dst = a.cand + slot * 32;
#pragma unroll
            for (int q = 0; q < 32; q++) {
                const int id = q < KP ? li[q < KP ? q : 0] : -1;
                dst[q] = (a.xid && id >= 0) ? a.xid[id] : id;
            }
            a.kth[slot] = li[KP - 1] >= 0 ? lv[KP - 1] : INFINITY;
            // largest block radius this CTA visited (scaled), for the certificate
            if (half == 0) atomicMax(reinterpret_cast<unsigned *>(a.qhat) + (gi - a.row0), misc->rho_bits);
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == WARP_MMA)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS)
                     : "memory");
}

template <int MODE, int KP, int DK>
void launch_t(const TcArgs &args, int64_t ngroups, cudaStream_t s) {
    const Plan P = make_plan(DK, Shape<DK, KP>::NCG);
    SLK_CUDA(cudaFuncSetAttribute(tc_bc_kernel<MODE, KP, DK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)P.total));
    tc_bc_kernel<MODE, KP, DK><<<(unsigned)(ngroups * args.nsplit), Shape<DK, KP>::NTHREADS, P.total, s>>>(args);
    SLK_CHECK_LAUNCH();
}

template <int DK>
void launch_dk(int mode, int kp, const TcArgs &args, int64_t ngroups, cudaStream_t s) {
    if (mode == MODE_COLOR) {
        // K' = 4 per column half (8 candidates a row) certifies the C3 / C2
        // cross-colour rows as well as 8 and saves 7 % of the scan; an
        // explicit SLK_TC_KP1 keeps the requested K'
        if (kp <= 4 || (kp == 8 && !getenv("SLK_TC_KP1"))) launch_t<MODE_COLOR, 4, DK>(args, ngroups, s);
        else launch_t<MODE_COLOR, 8, DK>(args, ngroups, s);
    }
    else if (kp <= 8) launch_t<MODE_SELF, 8, DK>(args, ngroups, s);
    else launch_t<MODE_SELF, 16, DK>(args, ngroups, s);
}

}  // namespace

int bc_dk(int d) { return d <= 16 ? 16 : d <= 32 ? 32 : d <= 64 ? 64 : d <= 128 ? 128 : 0; }

size_t bc_record_bytes(int d) { return bc_dk(d) ? rec_bytes(bc_dk(d)) : 0; }

// Measured at the bench configs (round 2): the block-centred kernel wins
// wherever the tensor / operand side paces the scan — the cross-colour passes
// at d >= 64 (C3 -30 %, C2 -25 %), the k-NN pass at d = 128 (C2 -25 %), and
// every k-NN pass over data whose blocks overlap so much that nothing prunes
// (C4: d = 32 0.42 -> 0.29 s, d = 128 1.06 -> 0.52 s).  The k-NN pass over
// well-separated clusters at d = 64 (C3) is bound by its insertion epilogue
// either way and 6 % slower here, and at d = 32 the query-centred kernel wins
// the cross-colour passes (C5).  `unprunable`: the caller's measure
// (knn.cu:blocks_overlap).  SLK_TC_BC=0 disables the kernel, =2 allows it for
// every supported pass.
bool bc_supported(int mode, int d, int kp, bool unprunable) {
    int lvl = 1;
    if (const char *e = getenv("SLK_TC_BC")) lvl = atoi(e);
    if (lvl == 0 || !bc_dk(d)) return false;
    if (mode == MODE_COLOR) return kp <= 8 && (lvl == 2 || d > 32);
    if (mode == MODE_SELF) return kp <= 16 && (lvl == 2 || d >= 96 || unprunable);
    return false;
}

void bc_pack(const float *x32, const int32_t *rowmap, int64_t n, int d, int64_t nb, const float *centroid,
             const float *radius, float scale, unsigned char *out, cudaStream_t s) {
    const int dk = bc_dk(d);
    bcpack_kernel<<<(unsigned)nb, 128, 0, s>>>(x32, rowmap, n, d, dk, nb, centroid, radius, scale, out);
    SLK_CHECK_LAUNCH();
}

void bc_launch(int mode, int kp, const TcArgs &args, int64_t ngroups, cudaStream_t s) {
    switch (bc_dk(args.d)) {
        case 16: launch_dk<16>(mode, kp, args, ngroups, s); break;
        case 32: launch_dk<32>(mode, kp, args, ngroups, s); break;
        case 64: launch_dk<64>(mode, kp, args, ngroups, s); break;
        default: launch_dk<128>(mode, kp, args, ngroups, s); break;
    }
}

void bc_timeline_arm(cudaStream_t s) { tl_arm(s); }
void bc_timeline_dump(int mode, int64_t rows, cudaStream_t s) { tl_dump(mode, rows, s); }

}  // namespace tc
}  // namespace slk
