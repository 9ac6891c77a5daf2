// tc_scan.cuh — host interface of the tcgen05 scan (tc_scan.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace slk {
namespace tc {

struct TcArgs {
    const float *qp;         // tc-packed queries [nqb][128 * dk] (knn.cu:tcpack_kernel)
    const float *xp;         // tc-packed index   [nxb][128 * dk]
    int64_t nq, nx;
    int d, dp, dk;           // dims, packed dims (multiple of 16), MMA K extent (k_extent)
    int64_t qb0;             // first query block of this launch
    const float *gcentroid;  // centring point of each query group of the launch, dims-major [dp][ngroups]
    int64_t ngroups;
    int64_t nqb_total;       // query blocks of the query set
    float scale;             // power of two applied after centring
    float inv_scale2;        // 1 / scale^2 (exact)
    const uint8_t *mask;
    const int32_t *qcolor;
    const int32_t *xcolor;   // MODE_COLOR: padded to whole 128-point blocks
    int32_t *cand;           // [rows][nsplit][32] (slots >= K' hold -1)
    float *kth;              // [rows][nsplit] approximate K'-th value (scaled units, rounded down)
    float *qhat;             // [rows] |q^|^2 (scaled units)
    int64_t row0, row1;
    const int32_t *sb_order;  // visit order (scan_common.cuh:BlockVisitor)
    const float *sb_lb;
    const float *flat_lb;
    const int32_t *nvalid;
    int64_t nsb;
    unsigned long long *tiles_done;
    const int32_t *qid;      // query row -> id in the index, -1 = padding (or null)
    int nsplit;              // CTAs per query block, each scanning 1/nsplit of the visit order
    const int32_t *xid;      // index position -> id written to cand (re-blocked index), or null
    int self_pos;            // MODE_SELF over one re-blocked set: a row's own point sits at its position
    int nprod;               // fp16 products per 16 dims: 1 (hi.hi) or 3 (hi.hi + hi.lo + lo.hi); see nprod_for
    const unsigned char *bcx;  // block-centred kernel (tc_bc.cu): bc-packed index records; qp = raw query rows
    const int32_t *xpos;     // block-centred kernel over a re-blocked index: id -> position (self exclusion), or null
};

// fp16 products per 16 dims for a pass: 3 (certificate
// slack 2^-22 relative to |q~||x~|); SLK_TC_NPROD=1 selects one product
// (2^-11) for every pass.
int nprod_for(bool rerun);
// Block-centred one-product kernel (tc_bc.cu): index
// converted once per call (bc_pack, bc_record_bytes per 128-point block),
// queries re-centred per tile into tensor memory; two column-half lists per
// row, the refine's certificate takes the largest visited block radius from
// qhat (float bits, zero-initialised).
bool bc_supported(int mode, int d, int kp, bool unprunable = false);
size_t bc_record_bytes(int d);
// rowmap (optional): position p of the index is row rowmap[p] of x32
void bc_pack(const float *x32, const int32_t *rowmap, int64_t n, int d, int64_t nb, const float *centroid,
             const float *radius, float scale, unsigned char *out, cudaStream_t s);
void bc_launch(int mode, int kp, const TcArgs &args, int64_t ngroups, cudaStream_t s);
void bc_timeline_arm(cudaStream_t s);
void bc_timeline_dump(int mode, int64_t rows, cudaStream_t s);
// diagnostic timeline probe (no-ops unless built with -DSLK_TIMELINE)
void timeline_arm(cudaStream_t s);
void timeline_dump(int mode, int64_t rows, cudaStream_t s);

// MMA K extent for d dims: d rounded up to 16, plus the augmented norm step
// when use_aug(d) (tc_scan.cu)
bool use_aug(int d);
// d > 128: chunked kernel (query hi term in TMEM, index blocks streamed in
// chunk_dims(d)-dim stages); k_extent(d) is then d rounded up to 64
bool chunked(int d);
int k_extent(int d);
// dims per contiguous sub-block of the tc-packed layout (= k_extent unless chunked)
int chunk_dims(int d);
size_t smem_bytes(int d);
bool supported(int d);
// Query blocks per CTA (1 or 2) for d dims and K' = kp.
int group_blocks(int d, int kp);
// kp: candidates kept per row (2..32; the certificate needs kp > k); qb query
// blocks per CTA sharing one centring point (group_blocks)
void launch(int mode, int kp, int qb, const TcArgs &args, int64_t ngroups, cudaStream_t s);
// One query block per CTA with two epilogue warps per TMEM lane quarter, each
// keeping a K' list over one half of every tile's columns: every CTA writes 2
// candidate lists per row (slot split * 2 + half).  k-NN (MODE_SELF, K' <= 16)
// and cross-colour (MODE_COLOR, K' <= 8) passes.
bool halves_supported(int mode, int d, int kp);
void launch_halves(int mode, int kp, const TcArgs &args, int64_t ngroups, cudaStream_t s);

}  // namespace tc
}  // namespace slk
