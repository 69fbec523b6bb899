// serial_bench.cu -- replay of the fixed-point decoder's single-warp band on real
// inputs (tools/ubench/serial_dump.py): every width-2048 node the band is handed
// while decoding frames of a BASELINE config, in decode order, through se::root
// exactly as sc_decode_kernel calls it (S = W = 2048), checked against the integer
// oracle's partial sums.  Reports cycles per frame spent inside the engine, per
// block, so that engine variants can be compared without the rest of the kernel.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
//          [-DSE_PROF] [-DSE_SP=true] [-DSE_W32_NPAT=n] [-D...] -o serial_bench serial_bench.cu
// run:   serial_bench data/serial_c3.bin [blocks=296] [threads=256] [reps=3]
#include <cuda_runtime.h>
#include <limits.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

#define PQ_CHECK(cond) ((void)0)
#define PQ_JITTER() ((void)0)
#ifndef PQ_WIDE_WARP_LOG2
#define PQ_WIDE_WARP_LOG2 11
#endif
__constant__ float CORR_TAB_C[4097];
#ifndef SE_SP
#define SE_SP false  // true: the pattern routines of the clustered kernels
#endif
#ifndef SE_HEADER
#define SE_HEADER "../../paper_1204_5882_b200/csrc/serial_q88.cuh"
#endif
#include SE_HEADER

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));     \
            exit(1);                                                                       \
        }                                                                                  \
    } while (0)

struct Rec {  // device views of one record
    int d0;
    uint32_t j;
    const int16_t *vals;
    const uint32_t *expect;
    const uint8_t *ty;
    const uint32_t *fm;
};

// optional i-cache pressure between nodes: ICF_KB KB of straight-line code the
// other warps execute while the serial warp is parked (as the block and upper
// bands do in the real kernel)
#ifndef ICF_REPS
#define ICF_REPS 0
#endif
__device__ __noinline__ float icache_filler(float x)
{
#pragma unroll
    for (int i = 0; i < 2048; i++) x = x * 1.0001f + (float)i;
    return x;
}

__global__ void __launch_bounds__(256, 2)
replay(const Rec *recs, int nodes, int frames, int wl, unsigned long long *cycles, unsigned *mism,
       unsigned long long *prof, float *sink)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t W = 1u << wl, S = W;
    float *st = (float *)smem_raw;              // [2S]
    uint32_t *xs = (uint32_t *)(st + 2 * S);    // [S/32]
    uint8_t *ty = (uint8_t *)(xs + S / 32);     // [2S]
    uint32_t *fm = (uint32_t *)(ty + 2 * S);    // [S/32]
    const int tid = threadIdx.x, nthr = blockDim.x;
    se::load_tables();
#ifdef SE_PROF
    if (tid < 32) ((unsigned long long *)se::se_prof)[tid] = 0;
#endif
    __syncthreads();
    const int frame = blockIdx.x % frames;
    unsigned long long total = 0;
    unsigned bad = 0;
    float fl = (float)tid;
    for (int i = 0; i < nodes; i++) {
        const Rec r = recs[frame * nodes + i];
        __syncthreads();
        for (uint32_t k = tid; k < W; k += nthr) st[k] = (float)r.vals[k];
        for (uint32_t k = tid; k < 2 * W; k += nthr) ty[k] = r.ty[k];
        for (uint32_t k = tid; k < W / 32; k += nthr) fm[k] = r.fm[k];
        __syncthreads();
        if (tid < 32) {
            const long long t0 = clock64();
            se::root<SE_SP>(st + 2 * S, xs, ty, fm, S, r.d0, r.d0, r.j);
            total += clock64() - t0;
        } else if (ICF_REPS) {
            for (int q = 0; q < ICF_REPS; q++) fl = icache_filler(fl);
        }
        __syncthreads();
        if (tid < 32)
            for (uint32_t k = tid; k < W / 32; k += 32) bad += xs[k] != r.expect[k];
    }
    if (tid == 0) cycles[blockIdx.x] = total;
    if (tid < 32) atomicAdd(mism, bad);
    if (fl == 12345.678f) sink[0] = fl;
#ifdef SE_PROF
    __syncthreads();
    if (blockIdx.x == 0 && tid < 32) prof[tid] = ((unsigned long long *)se::se_prof)[tid];
#endif
}

// the decoder's fixed-point tables (polarsc.cu fixed_tables, same construction)
static void fixed_tables(float *corr, int *taui)
{
    static int C[4097];
    for (int k = 0; k <= 4096; k++) {
        C[k] = (int)lrint(log1p(exp(-(double)k / 256.0)) * 256.0);
        corr[k] = (float)C[k];
    }
    std::vector<int> L(32768);
    for (int a = 0; a < 32768; a++) {
        int best = INT_MAX;
        if (2 * a >= 4096) best = C[4096] - C[0];
        else
            for (int d = 0; d <= 4096; d++) best = std::min(best, C[std::min(2 * a + d, 4096)] - C[d]);
        L[a] = std::max(0, a + best);
    }
    for (int a = 32766; a >= 0; a--) L[a] = std::min(L[a], L[a + 1]);
    auto chain = [&](int t, int k) {
        for (int i = 0; i < k; i++) t = L[t];
        return t;
    };
    for (int k = 0; k < 26; k++) {
        if (chain(32767, k) < 1) {
            taui[k] = INT_MAX;
            continue;
        }
        int lo = 0, hi = 32767;
        while (hi - lo > 1) {
            const int mid = (lo + hi) / 2;
            if (chain(mid, k) >= 1) hi = mid;
            else lo = mid;
        }
        taui[k] = hi;
    }
}

int main(int argc, char **argv)
{
    const char *path = argc > 1 ? argv[1] : "tools/ubench/data/serial_c3.bin";
    const int blocks = argc > 2 ? atoi(argv[2]) : 296;
    const int threads = argc > 3 ? atoi(argv[3]) : 256;
    const int reps = argc > 4 ? atoi(argv[4]) : 3;
    FILE *fh = fopen(path, "rb");
    if (!fh) {
        perror(path);
        return 1;
    }
    fseek(fh, 0, SEEK_END);
    const long sz = ftell(fh);
    fseek(fh, 0, SEEK_SET);
    std::vector<unsigned char> buf(sz);
    if (fread(buf.data(), 1, sz, fh) != (size_t)sz) return 1;
    fclose(fh);
    int hdr[4];
    memcpy(hdr, buf.data(), 16);
    const int n = hdr[0], wl = hdr[1], frames = hdr[2], nodes = hdr[3];
    const uint32_t W = 1u << wl;
    const size_t recsz = 8 + 2 * W + W / 8 + 2 * W + W / 8;
    if ((size_t)sz != 16 + recsz * frames * nodes) {
        fprintf(stderr, "bad file size\n");
        return 1;
    }
    unsigned char *d_buf;
    CK(cudaMalloc(&d_buf, sz));
    CK(cudaMemcpy(d_buf, buf.data(), sz, cudaMemcpyHostToDevice));
    std::vector<Rec> recs(frames * nodes);
    for (int i = 0; i < frames * nodes; i++) {
        const size_t off = 16 + recsz * i;
        memcpy(&recs[i].d0, &buf[off], 4);
        memcpy(&recs[i].j, &buf[off + 4], 4);
        recs[i].vals = (const int16_t *)(d_buf + off + 8);
        recs[i].expect = (const uint32_t *)(d_buf + off + 8 + 2 * W);
        recs[i].ty = d_buf + off + 8 + 2 * W + W / 8;
        recs[i].fm = (const uint32_t *)(d_buf + off + 8 + 2 * W + W / 8 + 2 * W);
    }
    Rec *d_recs;
    CK(cudaMalloc(&d_recs, recs.size() * sizeof(Rec)));
    CK(cudaMemcpy(d_recs, recs.data(), recs.size() * sizeof(Rec), cudaMemcpyHostToDevice));
    static float corr[4097];
    int taui[26];
    fixed_tables(corr, taui);
    CK(cudaMemcpyToSymbol(CORR_TAB_C, corr, sizeof corr));
    CK(cudaMemcpyToSymbol(se::TAUI, taui, sizeof taui));
    unsigned long long *d_cyc, *d_prof;
    unsigned *d_mism;
    float *d_sink;
    CK(cudaMalloc(&d_cyc, blocks * sizeof(unsigned long long)));
    CK(cudaMalloc(&d_prof, 32 * sizeof(unsigned long long)));
    CK(cudaMalloc(&d_mism, 4));
    CK(cudaMalloc(&d_sink, 4));
    CK(cudaMemset(d_prof, 0, 32 * sizeof(unsigned long long)));
    const size_t smem = 8 * W + W / 8 + 2 * W + W / 8;
    CK(cudaFuncSetAttribute(replay, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    printf("%s: n=%d W=%u frames=%d nodes/frame=%d blocks=%d threads=%d icf=%d\n", path, n, W, frames, nodes, blocks,
           threads, ICF_REPS);
    for (int rep = 0; rep < reps; rep++) {
        CK(cudaMemset(d_mism, 0, 4));
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        replay<<<blocks, threads, smem>>>(d_recs, nodes, frames, wl, d_cyc, d_mism, d_prof, d_sink);
        cudaEventRecord(b);
        CK(cudaDeviceSynchronize());
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        std::vector<unsigned long long> cyc(blocks);
        unsigned mism;
        CK(cudaMemcpy(cyc.data(), d_cyc, blocks * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(&mism, d_mism, 4, cudaMemcpyDeviceToHost));
        std::sort(cyc.begin(), cyc.end());
        printf("rep %d: kernel %.3f ms; engine cycles/frame min %llu median %llu max %llu; mismatching words %u\n", rep, ms,
               cyc.front(), cyc[blocks / 2], cyc.back(), mism);
    }
#ifdef SE_PROF
    unsigned long long prof[32];
    CK(cudaMemcpy(prof, d_prof, sizeof prof, cudaMemcpyDeviceToHost));
    const char *names[16] = {"child8", "w16", "w32", "walk", "s4", "s5", "s6", "s7", "s8", "s9", "s10", "s11", "s12", "s13", "s14", "s15"};
    for (int s = 0; s < 16; s++)
        if (prof[16 + s])
            printf("  slot %-7s calls %8llu cycles %10llu  (%.0f / call; block 0, all reps, inclusive)\n", names[s], prof[16 + s],
                   prof[s], (double)prof[s] / prof[16 + s]);
#endif
    return 0;
}
