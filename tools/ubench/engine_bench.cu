// Microbenchmarks of the decoder's building blocks (includes the product source).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 -I../../include -o engine_bench engine_bench.cu
#define PQ_UBENCH_TIMING 1
#include "../../paper_1204_5882_b200/csrc/polarsc.cu"

__global__ void k_f_latency(const float *in, float *out, int iters, long long *cyc)
{
    load_log_table();
    __syncthreads();
    float a = in[threadIdx.x], b = in[threadIdx.x + 32];
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        a = pq_f<PQ_F_EXACT>(a, b) + 0.5f;
        b = b * 1.0001f;
    }
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int ILP>
__global__ void k_f_ilp(const float *in, float *out, int iters, long long *cyc)
{
    load_log_table();
    __syncthreads();
    float a[ILP], b = in[threadIdx.x + 32];
#pragma unroll
    for (int k = 0; k < ILP; k++) a[k] = in[(threadIdx.x + k) & 31];
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int k = 0; k < ILP; k++) a[k] = pq_f<PQ_F_EXACT>(a[k], b) + 0.5f;
        b = b * 1.0001f;
    }
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int k = 0; k < ILP; k++) s += a[k];
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_shfl_latency(const float *in, float *out, int iters, long long *cyc)
{
    float a = in[threadIdx.x];
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) a = __shfl_sync(0xffffffffu, a, (threadIdx.x + 1) & 31) + 1.0f;
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

// one warp, repeated engine32 on a W=32 sub-tree whose local heap types are ty[1..63]
__global__ void k_engine(const float *in, const uint8_t *ty_g, float *out, int iters, int plain, long long *cyc)
{
    __shared__ uint8_t ty[64];
    load_log_table();
    for (int i = threadIdx.x; i < 64; i += 32) ty[i] = ty_g[i];
    __syncthreads();
    WarpCtx c;
    c.ty = ty;
    c.dump = nullptr;
    c.N = 32;
    c.plain = plain;
    c.dS = 0;
    c.jS = 0;
    c.prof = nullptr;
    float v = in[threadIdx.x];
    uint32_t acc = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        acc ^= engine32<PQ_F_EXACT>(v, 1, 32, c);
        v = v + 0.001f * (float)(acc & 1u);
    }
    long long t1 = clock64();
    out[threadIdx.x] = v + (float)acc;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

// one warp decodes the four W=256 sub-trees of the c1 code (S = N = 1024)
// through the product's warp_walk, from shared-memory stage buffers
template <int FM>
__global__ void k_c1_warp(const uint8_t *types_g, const float *llr, long long *cyc, uint32_t *out, int reps)
{
    __shared__ uint8_t ty[2048];
    __shared__ float st[2048];
    __shared__ uint32_t xs[32];
    load_log_table();
    for (int i = threadIdx.x; i < 2048; i += 32) ty[i] = types_g[i];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    long long t0 = clock64();
    for (int rep = 0; rep < reps; rep++)
        for (int sI = 0; sI < 4; sI++) {
            // stage buffer for width 256 lives at st_end - 512
            for (int q = 0; q < 8; q++) st[2048 - 512 + 32 * q + lane] = llr[256 * sI + 32 * q + lane] + 0.001f * (float)rep;
            __syncwarp();
            warp_walk<FM>(st + 2048, xs, ty, nullptr, 1024, 1024, 0, 0, 0, 2, (uint32_t)sI);
        }
    long long t1 = clock64();
    out[blockIdx.x * 32 + lane] = xs[lane];
    if (lane == 0 && blockIdx.x == 0) cyc[0] = (t1 - t0) / reps;
}

int main()
{
    float h[64];
    for (int i = 0; i < 64; i++) h[i] = 0.3f + 0.37f * (i % 13) - 1.5f * (i % 3 == 0);
    float *in, *out;
    long long *cyc, c;
    uint8_t *ty;
    cudaMalloc(&in, 256);
    cudaMalloc(&out, 256);
    cudaMalloc(&cyc, 8);
    cudaMalloc(&ty, 64);
    cudaMemcpy(in, h, 256, cudaMemcpyHostToDevice);
    const int iters = 2000;
    for (int r = 0; r < 2; r++) k_f_latency<<<1, 32>>>(in, out, iters, cyc);
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("f latency: %.1f cycles\n", (double)c / iters);
    for (int r = 0; r < 2; r++) k_f_ilp<2><<<1, 32>>>(in, out, iters, cyc);
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("f x2 ILP: %.1f cycles per iteration\n", (double)c / iters);
    for (int r = 0; r < 2; r++) k_f_ilp<4><<<1, 32>>>(in, out, iters, cyc);
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("f x4 ILP: %.1f cycles per iteration\n", (double)c / iters);
    for (int r = 0; r < 2; r++) k_f_ilp<8><<<1, 32>>>(in, out, iters, cyc);
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("f x8 ILP: %.1f cycles per iteration\n", (double)c / iters);
    for (int r = 0; r < 2; r++) k_shfl_latency<<<1, 32>>>(in, out, iters, cyc);
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("shfl+add latency: %.1f cycles\n", (double)c / iters);
    // plain: all 31 internal nodes mixed, leaves: alternate frozen/info
    uint8_t t[64];
    for (int i = 0; i < 64; i++) t[i] = i < 32 ? NT_MIXED : ((i & 1) ? NT_RATE1 : NT_RATE0);
    cudaMemcpy(ty, t, 64, cudaMemcpyHostToDevice);
    for (int r = 0; r < 2; r++) k_engine<<<1, 32>>>(in, ty, out, 200, 1, cyc);
    {
        unsigned long long z[16] = {0};
        cudaMemcpyToSymbol(g_ub_time, z, sizeof z);
        cudaMemcpyToSymbol(g_ub_count, z, sizeof z);
    }
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("engine32 plain (31 mixed nodes): %.0f cycles/call = %.1f per node\n", (double)c / 200, (double)c / 200 / 31);
    {
        uint8_t *tyh = (uint8_t *)malloc(2048);
        FILE *fp = fopen("tools/ubench/c1_types.bin", "rb");
        if (fp) {
            if (fread(tyh, 1, 2048, fp) != 2048) return 1;
            fclose(fp);
            float *lh = (float *)malloc(4096);
            uint32_t seed = 1;
            for (int i = 0; i < 1024; i++) {
                seed = seed * 1664525u + 1013904223u;
                lh[i] = ((seed >> 8) & 1 ? 1.0f : -1.0f) * (0.5f + 3.0f * ((seed >> 9) & 1023) / 1023.0f);
            }
            float *dl;
            uint8_t *dty;
            uint32_t *dout;
            cudaMalloc(&dl, 4096);
            cudaMalloc(&dty, 2048);
            cudaMalloc(&dout, 148 * 128);
            cudaMemcpy(dl, lh, 4096, cudaMemcpyHostToDevice);
            cudaMemcpy(dty, tyh, 2048, cudaMemcpyHostToDevice);
            for (int r = 0; r < 2; r++) k_c1_warp<PQ_F_MINSUM><<<1, 32>>>(dty, dl, cyc, dout, 10);
            cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            printf("c1 warp levels, MIN-SUM f: %lld cycles\n", c);
            for (int r = 0; r < 2; r++) k_c1_warp<PQ_F_EXACT><<<1, 32>>>(dty, dl, cyc, dout, 10);
            k_c1_warp<PQ_F_EXACT><<<1, 32>>>(dty, dl, cyc, dout, 1);
            cudaDeviceSynchronize();
            cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            printf("c1 warp levels (4 x W256 sub-trees): %lld cycles\n", c);
            unsigned long long tt[16], cc[16];
            cudaMemcpyFromSymbol(tt, g_ub_time, sizeof tt);
            cudaMemcpyFromSymbol(cc, g_ub_count, sizeof cc);
            k_c1_warp<PQ_F_EXACT><<<148, 32>>>(dty, dl, cyc, dout, 10);  // the launch ncu profiles
            cudaDeviceSynchronize();
            printf("dec8: %llu calls %.0f cycles/call; dec32: %llu calls %.0f cycles/call\n", cc[0],
                   (double)tt[0] / (cc[0] ? cc[0] : 1), cc[1], (double)tt[1] / (cc[1] ? cc[1] : 1));
        }
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
