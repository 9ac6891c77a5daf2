// tc_scan.cuh — host interface of the tcgen05 scan (tc_scan.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace slk {
namespace tc {

struct TcArgs {
    const float *qp;         // packed queries [nqb][dp][128]
    const float *xp;         // packed index   [nxb][dp][128]
    int64_t nq, nx;
    int d, dp, dk;           // dims, packed dims (multiple of 16), MMA K extent
    int64_t qb0;             // first query block of this launch
    const float *qcentroid;  // query block centroids, dims-major [dp][nqb_total]
    int64_t nqb_total;
    float scale;             // power of two applied after centring
    float inv_scale2;        // 1 / scale^2 (exact)
    const uint8_t *mask;
    const int32_t *qcolor, *xcolor;
    int32_t *cand;           // [rows][32R]
    float *kth;              // [rows] approximate K'-th value (scaled units)
    float *qhat;             // [rows] |q^|^2 (scaled units)
    int64_t row0, row1;
    const int32_t *sb_order;
    const float *sb_key;
    const float *sb_lb;
    const float *blk_lb;
    int64_t nsb;
    unsigned long long *tiles_done;
    const int32_t *qid;      // query row -> id in the index, -1 = padding (or null)
};

size_t smem_bytes(int d, int R);
bool supported(int d, int R);
void launch(int mode, int R, const TcArgs &args, int64_t nqb, cudaStream_t s);

}  // namespace tc
}  // namespace slk
