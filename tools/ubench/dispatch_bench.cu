// Interpreter dispatch cost on sm_100a: uniform byte-code loop, one warp.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k_dispatch(const uint8_t *prog_g, int len, int reps, long long *cyc, float *out)
{
    __shared__ uint8_t prog[4096];
    for (int i = threadIdx.x; i < len; i += 32) prog[i] = prog_g[i];
    __syncwarp();
    float x = threadIdx.x * 0.1f, y = 1.0f;
    const int lane = threadIdx.x & 31;
    long long t0 = clock64();
    for (int r = 0; r < reps; r++) {
        uint32_t nxt = prog[0];
        for (int pc = 0; pc < len; pc++) {
            uint32_t op;
            if (MODE == 1) {  // prefetch the next op
                op = nxt;
                nxt = prog[pc + 1];
            } else {
                op = prog[pc];
            }
            switch (op & 7u) {
            case 0: x = x + y; break;
            case 1: x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31); break;
            case 2: y = y * 1.0001f; break;
            case 3: x = x - y; break;
            case 4: y = __shfl_down_sync(0xffffffffu, y, 1) + 1.0f; break;
            case 5: x = fmaxf(x, y); break;
            case 6: x = x * 0.5f; break;
            default: y = y + 1.0f; break;
            }
        }
    }
    long long t1 = clock64();
    out[threadIdx.x] = x + y;
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) / ((long long)reps * len);
}

__global__ void k_branchchain(int iters, long long *cyc, float *out, uint32_t seed)
{
    // uniform data-dependent if-chains (like type checks)
    float x = threadIdx.x;
    uint32_t s = seed;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        s = s * 1664525u + 1013904223u;
        const uint32_t t = (s >> 13) & 3u;
        if (t == 0) x += 1.0f;
        else if (t == 1) x *= 1.0001f;
        else if (t == 2) x -= 0.5f;
        else x = x * 0.999f + 1.0f;
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) / iters;
}

int main()
{
    uint8_t h[4096];
    uint32_t s = 7;
    for (int i = 0; i < 4096; i++) {
        s = s * 1664525u + 1013904223u;
        h[i] = (s >> 20) & 7;
    }
    uint8_t *dp;
    long long *cyc, c;
    float *out;
    cudaMalloc(&dp, 4096);
    cudaMalloc(&cyc, 8);
    cudaMalloc(&out, 128);
    cudaMemcpy(dp, h, 4096, cudaMemcpyHostToDevice);
    for (int r = 0; r < 2; r++) k_dispatch<0><<<1, 32>>>(dp, 1000, 20, cyc, out);
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("switch dispatch, LDS op per iteration:      %lld cycles/op\n", c);
    for (int r = 0; r < 2; r++) k_dispatch<1><<<1, 32>>>(dp, 1000, 20, cyc, out);
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("switch dispatch, op prefetched:              %lld cycles/op\n", c);
    for (int r = 0; r < 2; r++) k_branchchain<<<1, 32>>>(100000, cyc, out, 5);
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("uniform if-chain on computed value:          %lld cycles/iter\n", c);
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
