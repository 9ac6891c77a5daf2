// scan_common.cuh — device pieces shared by the two distance-scan kernels
// (exact-fp32 FFMA scan in knn.cu, tcgen05 tensor-core scan in tc_scan.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace slk {
namespace scan {

constexpr int BM = 128;   // query rows per CTA
constexpr int BN = 128;   // index points per block
constexpr int KC = 16;    // dims per operand chunk
constexpr int NT = 256;   // threads per CTA
constexpr int CAP = 32;   // per-row candidate buffer
constexpr unsigned FULL = 0xffffffffu;

enum Mode { MODE_NONE = 0, MODE_MASK = 1, MODE_COLOR = 2, MODE_SELF = 3 };

// --------------------------------------------------- warp sorted lists
// A warp holds a sorted list of 32R (value, id) pairs, element p = r*32+lane,
// ascending by (value, id).  Insertion shifts the suffix right by one.
template <class V>
__device__ __forceinline__ bool pair_gt(V av, int ai, V bv, int bi) {
    return av > bv || (av == bv && ai > bi);
}

template <int R, class V>
__device__ __forceinline__ void warp_list_insert(V (&lv)[R], int (&li)[R], V v, int id, int lane) {
    bool g[R];
    V pv[R];
    int pi[R];
    bool pg[R];
    V tv[R];
    int ti[R];
    bool tg[R];
#pragma unroll
    for (int r = 0; r < R; r++) {
        g[r] = pair_gt(lv[r], li[r], v, id);
        pv[r] = __shfl_up_sync(FULL, lv[r], 1);
        pi[r] = __shfl_up_sync(FULL, li[r], 1);
        pg[r] = __shfl_up_sync(FULL, (int)g[r], 1) != 0;
        tv[r] = __shfl_sync(FULL, lv[r], 31);
        ti[r] = __shfl_sync(FULL, li[r], 31);
        tg[r] = __shfl_sync(FULL, (int)g[r], 31) != 0;
    }
#pragma unroll
    for (int r = 0; r < R; r++) {
        if (lane == 0) {
            if (r == 0) {
                pg[r] = false;
            } else {
                pv[r] = tv[r - 1];
                pi[r] = ti[r - 1];
                pg[r] = tg[r - 1];
            }
        }
        if (g[r]) {
            if (pg[r]) {
                lv[r] = pv[r];
                li[r] = pi[r];
            } else {
                lv[r] = v;
                li[r] = id;
            }
        }
    }
}

// Bitonic sort of the 32R warp-distributed pairs, ascending by (value, id).
template <int R, class V>
__device__ __forceinline__ void warp_bitonic_sort(V (&lv)[R], int (&li)[R], int lane) {
    constexpr int N = 32 * R;
#pragma unroll
    for (int size = 2; size <= N; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            if (stride >= 32) {
                int rs = stride / 32;
#pragma unroll
                for (int r = 0; r < R; r++) {
                    int partner = r ^ rs;
                    if (partner > r) {
                        int p = r * 32 + lane;
                        bool up = (p & size) == 0;
                        bool sw = up ? pair_gt(lv[r], li[r], lv[partner], li[partner])
                                     : pair_gt(lv[partner], li[partner], lv[r], li[r]);
                        if (sw) {
                            V tv = lv[r];
                            int ti = li[r];
                            lv[r] = lv[partner];
                            li[r] = li[partner];
                            lv[partner] = tv;
                            li[partner] = ti;
                        }
                    }
                }
            } else {
#pragma unroll
                for (int r = 0; r < R; r++) {
                    int p = r * 32 + lane;
                    V ov = __shfl_xor_sync(FULL, lv[r], stride);
                    int oi = __shfl_xor_sync(FULL, li[r], stride);
                    bool lower = (lane & stride) == 0;
                    bool up = (p & size) == 0;
                    // lower element keeps the min when ascending
                    bool mine_gt = pair_gt(lv[r], li[r], ov, oi);
                    bool take = (lower == up) ? mine_gt : !mine_gt;
                    if (take && !(lv[r] == ov && li[r] == oi)) {
                        lv[r] = ov;
                        li[r] = oi;
                    }
                }
            }
        }
    }
}

// Sorts a bitonic sequence of 32R warp-distributed pairs ascending
// (half-cleaner cascade: strides 16R .. 1).
template <int R, class V>
__device__ __forceinline__ void warp_bitonic_merge(V (&lv)[R], int (&li)[R], int lane) {
#pragma unroll
    for (int stride = 16 * R; stride > 0; stride >>= 1) {
        if (stride >= 32) {
            const int rs = stride / 32;
#pragma unroll
            for (int r = 0; r < R; r++) {
                const int partner = r ^ rs;
                if (partner > r && pair_gt(lv[r], li[r], lv[partner], li[partner])) {
                    V tv = lv[r];
                    int ti = li[r];
                    lv[r] = lv[partner];
                    li[r] = li[partner];
                    lv[partner] = tv;
                    li[partner] = ti;
                }
            }
        } else {
#pragma unroll
            for (int r = 0; r < R; r++) {
                V ov = __shfl_xor_sync(FULL, lv[r], stride);
                int oi = __shfl_xor_sync(FULL, li[r], stride);
                const bool lower = (lane & stride) == 0;
                const bool mine_gt = pair_gt(lv[r], li[r], ov, oi);
                if (lower ? mine_gt : pair_gt(ov, oi, lv[r], li[r])) {
                    lv[r] = ov;
                    li[r] = oi;
                }
            }
        }
    }
}

// Keeps in the sorted list L (32R pairs) the 32R smallest of L and the
// sorted batch B (32CB pairs): the top registers of L meet B reversed
// (elementwise min), which leaves a bitonic sequence holding exactly those,
// then one bitonic merge.  ~(log2 32R) shuffle stages instead of one
// insertion per candidate.
template <int R, int CB, class V>
__device__ __forceinline__ void warp_merge_batch(V (&lv)[R], int (&li)[R], V (&bv)[CB],
                                                 int (&bi)[CB], int lane) {
    constexpr int M = CB < R ? CB : R;  // only the smallest 32R of B can survive
#pragma unroll
    for (int q = 0; q < M; q++) {
        const int r = R - 1 - q;  // list register meeting batch register q, reversed
        V ov = __shfl_sync(FULL, bv[q], 31 - lane);
        int oi = __shfl_sync(FULL, bi[q], 31 - lane);
        if (pair_gt(lv[r], li[r], ov, oi)) {
            lv[r] = ov;
            li[r] = oi;
        }
    }
    warp_bitonic_merge<R>(lv, li, lane);
}

// Iterates the index blocks a query block must visit.  The
// visit order: superblocks (32 index blocks) in ascending centroid distance
// from the query block (its own cluster first, so row thresholds tighten
// before distant blocks come up); within a superblock, its members in id
// order.  Per query block the builder stores, in that order, each
// superblock's id and lower bound (sb_order, sb_lb: [nsb]) and its 32 member
// bounds (lb: [nsb][32]); +inf marks padding and same-coloured pairs, and
// superblocks past `nvalid` are never admissible.  A superblock or member
// whose bound exceeds the current largest row threshold is skipped
// (thresholds only fall, so skipping stays exact).
//
// Latency hiding: superblock bounds are read 32 at a time (one coalesced load
// per lane, ballot), the next 32 are prefetched, and the member bounds of the
// next PF admissible superblocks are kept in flight in static register slots
// (a load is only waited on when its slot is consumed).  Control flow is
// warp-uniform given a warp-uniform threshold.  With nsplit > 1 the
// positions are dealt round-robin over nsplit CTAs (small launches).
struct BlockVisitor {
    static constexpr int PF = 4;
    const int32_t *sb_order;
    const float *sb_lb;
    const float *lb;
    int nvalid;
    int split = 0, nsplit = 1;  // this CTA takes superblock positions p = split (mod nsplit)
    int base = 0;             // next chunk of 32 superblock positions to take
    unsigned sbmask = 0;      // admissible positions of the current chunk
    int cbase = 0;            // first position of the current chunk
    float c_lb = INFINITY;    // this lane's superblock bound in the current chunk
    float n_lb = INFINITY;    // ... in the prefetched next chunk
    int nq = 0, qh = 0;       // member-bound slots in flight, head slot
    int q_sb[PF];
    float q_lb[PF];
    unsigned bmask = 0;
    int cur_sb = 0;
    float my_lb = INFINITY;

    __device__ BlockVisitor(const int32_t *order, const float *sblb, const float *lbs, int nv, int lane,
                            int split_ = 0, int nsplit_ = 1)
        : sb_order(order), sb_lb(sblb), lb(lbs), nvalid(nv), split(split_), nsplit(nsplit_) {
        n_lb = lane < nvalid ? __ldg(sb_lb + lane) : INFINITY;
    }
    // next admissible superblock position, or -1
    __device__ __forceinline__ int pop_position(float thr, int lane) {
        while (!sbmask) {
            if (base >= nvalid) return -1;
            cbase = base;
            c_lb = n_lb;
            base += 32;
            n_lb = base + lane < nvalid ? __ldg(sb_lb + base + lane) : INFINITY;
            sbmask = __ballot_sync(0xffffffffu, c_lb != INFINITY && !(c_lb > thr) &&
                                                    (nsplit == 1 || (cbase + lane) % nsplit == split));
        }
        const int i = __ffs(sbmask) - 1;
        sbmask &= sbmask - 1;
        return cbase + i;
    }
    template <int I>
    __device__ __forceinline__ void put(int pos, int lane) {
        q_sb[I] = __ldg(sb_order + pos);
        q_lb[I] = __ldg(lb + (int64_t)pos * 32 + lane);
    }
    __device__ __forceinline__ void fill(float thr, int lane) {
        while (nq < PF) {
            const int pos = pop_position(thr, lane);
            if (pos < 0) return;
            switch ((qh + nq) & (PF - 1)) {
                case 0: put<0>(pos, lane); break;
                case 1: put<1>(pos, lane); break;
                case 2: put<2>(pos, lane); break;
                default: put<3>(pos, lane); break;
            }
            nq++;
        }
    }
    template <int I>
    __device__ __forceinline__ void take() {
        cur_sb = q_sb[I];
        my_lb = q_lb[I];
    }
    __device__ int64_t next(float thr, int lane) {
        while (true) {
            if (bmask) {
                const int m = __ffs(bmask) - 1;
                bmask &= bmask - 1;
                if (__shfl_sync(0xffffffffu, my_lb, m) > thr) continue;
                return (int64_t)cur_sb * 32 + m;
            }
            fill(thr, lane);
            if (nq == 0) return -1;
            switch (qh) {
                case 0: take<0>(); break;
                case 1: take<1>(); break;
                case 2: take<2>(); break;
                default: take<3>(); break;
            }
            qh = (qh + 1) & (PF - 1);
            nq--;
            bmask = __ballot_sync(0xffffffffu, my_lb != INFINITY && !(my_lb > thr));
        }
    }
};

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

}  // namespace scan
}  // namespace slk
