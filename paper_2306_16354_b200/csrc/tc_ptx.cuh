// tc_ptx.cuh — PTX wrappers shared by the tcgen05 scan kernels (tc_scan.cu,
// tc_bc.cu): mbarriers, UMMA descriptors and issue, TMEM loads/stores, bulk
// copies, and the diagnostic timeline probe.  Included inside
// namespace slk::tc::<anonymous> of each translation unit.
#pragma once

// ------------------------------------------------------------ timeline probe
// Diagnostic build only (-DSLK_TIMELINE, build.py variant "timeline"): each
// warp role stamps clock64() at its hand-offs for the first TL_IT tiles of
// CTAs 0..TL_CTAS-1; tc_pass dumps them (SLK_TIMELINE=<file>).
#ifdef SLK_TIMELINE
constexpr int TL_CTAS = 16, TL_EV = 16, TL_IT = 512;
__device__ unsigned long long *g_tl;  // one per translation unit
// epilogue counters of the same build: [0] 32-column chunks read per warp,
// [1] chunks with a passing column, [2] insertion-loop iterations per warp
// (divergent: max over lanes), [3] candidates examined per thread, [4] inserted
__device__ unsigned long long g_cnt[8];
#define TLC(i, v) atomicAdd(&g_cnt[i], (unsigned long long)(v))
#define TL(ev, it)                                                                                  \
    do {                                                                                            \
        if (g_tl && blockIdx.x < TL_CTAS && (it) < TL_IT)                                           \
            g_tl[((size_t)blockIdx.x * TL_EV + (ev)) * TL_IT + (it)] = clock64();                   \
    } while (0)
#else
#define TL(ev, it) \
    do {           \
    } while (0)
#define TLC(i, v) \
    do {          \
    } while (0)
#endif

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
#ifdef SLK_WATCHDOG
__device__ void watchdog_dump(int tag, int it, uint32_t parity, unsigned long long st);
#endif
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity, int tag = 0, int it = 0) {
    uint32_t done;
#ifdef SLK_WATCHDOG
    long long spins = 0;
#endif
    do {
        // suspend-time hint: the waiting warp sleeps in hardware until the phase
        // completes (or 0.1 ms passes) instead of spinning on issue slots the
        // working warps of its SM sub-partition need
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity), "r"(100000u)
            : "memory");
#ifdef SLK_WATCHDOG
        if (!done && ++spins == (1ll << 24)) {
            unsigned long long st;
            asm volatile("ld.shared.b64 %0, [%1];" : "=l"(st) : "r"(smem_u32(bar)));
            watchdog_dump(tag, it, parity, st);
        }
#endif
    } while (!done);
}
// spin form (no suspend hint): for a warp on the critical path whose
// barrier usually completes within a few hundred cycles
__device__ __forceinline__ void mbar_wait_spin(uint64_t *bar, uint32_t parity) {
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

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
        "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
        "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
        "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}
// Warp-collective forms for the MMA warp: every lane runs the issue loop and
// elect.sync picks one lane (always the same: the lowest active one) to issue,
// so ptxas emits no per-instruction ELECT retry loop around a divergent issue.
__device__ __forceinline__ void umma_f16_w(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(IDESC), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_f16_ta_w(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(b), "r"(IDESC), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_commit_w(uint64_t *bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
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

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; i++) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_ld(uint32_t taddr, float (&v)[32]) { tmem_ld32(taddr, v); }
__device__ __forceinline__ void tmem_ld(uint32_t taddr, float (&v)[16]) { tmem_ld16(taddr, v); }

// Two-term fp16 split of a centred, scaled pair: v ~ hi + lo with
// |hi + lo - v| <= 2^-22 |v| + 2^-25 per component (lo = fp16(v - hi), v - hi
// exact in fp32).  nrm accumulates |v|^2 of the unsplit fp32 values: the
// certificate (knn.cu:certified_floor_tc) charges the difference to the
// represented |hi + lo|^2 (<= 2^-21 |v|^2 + 2^-24 sqrt(d) |v|), which saves
// unpacking lo and forming hi + lo.
__device__ __forceinline__ void split2(float v0, float v1, __half2 &hi, __half2 &lo, float &nrm) {
    hi = __floats2half2_rn(v0, v1);
    const float2 fh = __half22float2(hi);
    lo = __floats2half2_rn(__fsub_rn(v0, fh.x), __fsub_rn(v1, fh.y));
    nrm = __fmaf_rn(v0, v0, nrm);
    nrm = __fmaf_rn(v1, v1, nrm);
}

// ------------------------------------------------------------ PTX: TMA bulk
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}


// SLK_TIMELINE=<file>: arm the probe before a scan launch, append the stamps after it
#ifdef SLK_TIMELINE
static unsigned long long *tl_buf = nullptr;
static void tl_arm(cudaStream_t s) {
    if (!getenv("SLK_TIMELINE")) return;
    const size_t bytes = sizeof(unsigned long long) * TL_CTAS * TL_EV * TL_IT;
    if (!tl_buf) SLK_CUDA(cudaMalloc(&tl_buf, bytes));
    SLK_CUDA(cudaMemsetAsync(tl_buf, 0, bytes, s));
    const unsigned long long zc[8] = {};
    SLK_CUDA(cudaMemcpyToSymbolAsync(g_cnt, zc, sizeof(zc), 0, cudaMemcpyHostToDevice, s));
    SLK_CUDA(cudaMemcpyToSymbolAsync(g_tl, &tl_buf, sizeof(tl_buf), 0, cudaMemcpyHostToDevice, s));
}
static void tl_dump(int mode, int64_t rows, cudaStream_t s) {
    const char *path = getenv("SLK_TIMELINE");
    if (!path || !tl_buf) return;
    const size_t n = (size_t)TL_CTAS * TL_EV * TL_IT;
    unsigned long long *h = (unsigned long long *)malloc(n * sizeof(unsigned long long));
    SLK_CUDA(cudaMemcpyAsync(h, tl_buf, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    SLK_CUDA(cudaStreamSynchronize(s));
    unsigned long long *z = nullptr;
    SLK_CUDA(cudaMemcpyToSymbol(g_tl, &z, sizeof(z)));
    unsigned long long c[8];
    SLK_CUDA(cudaMemcpyFromSymbol(c, g_cnt, sizeof(c)));
    fprintf(stderr, "[slk] epilogue counters mode %d rows %lld: chunks %llu hit %llu loop_iters %llu examined %llu inserted %llu\n",
            mode, (long long)rows, c[0], c[1], c[2], c[3], c[4]);
    FILE *f = fopen(path, "ab");
    if (f) {
        const long long hdr[5] = {mode, rows, TL_CTAS, TL_EV, TL_IT};
        fwrite(hdr, sizeof(hdr), 1, f);
        fwrite(h, sizeof(unsigned long long), n, f);
        fclose(f);
    }
    free(h);
}
#else
static void tl_arm(cudaStream_t) {}
static void tl_dump(int, int64_t, cudaStream_t) {}
#endif

