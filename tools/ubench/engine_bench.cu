// Microbenchmarks of the decoder's building blocks (includes the product source).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 -I../../include -o engine_bench engine_bench.cu
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
    for (int r = 0; r < 2; r++) k_shfl_latency<<<1, 32>>>(in, out, iters, cyc);
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("shfl+add latency: %.1f cycles\n", (double)c / iters);
    // plain: all 31 internal nodes mixed, leaves: alternate frozen/info
    uint8_t t[64];
    for (int i = 0; i < 64; i++) t[i] = i < 32 ? NT_MIXED : ((i & 1) ? NT_RATE1 : NT_RATE0);
    cudaMemcpy(ty, t, 64, cudaMemcpyHostToDevice);
    for (int r = 0; r < 2; r++) k_engine<<<1, 32>>>(in, ty, out, 200, 1, cyc);
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("engine32 plain (31 mixed nodes): %.0f cycles/call = %.1f per node\n", (double)c / 200, (double)c / 200 / 31);
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
