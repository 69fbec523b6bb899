// Latency of the serial band's primitives on one warp (cycles per dependent op).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 -DNO_UB -I../../include -o prim_bench prim_bench.cu
#include <cstdio>
#include "../../paper_1204_5882_b200/csrc/polarsc.cu"

template <int OP>
__global__ void k_prim(const float *in, float *out, int iters, long long *cyc)
{
    for (int i = threadIdx.x; i < 4097; i += blockDim.x) pq_corrtab[i] = CORR_TAB_C[i];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    float a = in[lane], b = in[lane + 32];
    uint32_t u = lane;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        if (OP == 0) a = pq_f<PQ_F_FIXED>(a, b);                         // fixed f
        if (OP == 1) a = __shfl_sync(0xffffffffu, a, (lane + 1) & 31);    // shfl idx
        if (OP == 2) a = __shfl_down_sync(0xffffffffu, a, 8);            // shfl down
        if (OP == 3) u = __ballot_sync(0xffffffffu, (u >> lane) & 1u) + u;  // ballot
        if (OP == 4) u = __all_sync(0xffffffffu, u & 1u) + u;            // vote.all
        if (OP == 5) u = __reduce_min_sync(0xffffffffu, u) + 1u;         // redux min
        if (OP == 6) a = qadd<PQ_F_FIXED>(a, b);                         // saturating add
        if (OP == 7) a = pq_gt<PQ_F_FIXED>(a, b, u & 1u);                // g
        if (OP == 8) a = pq_corrtab[(__float_as_uint(a) & 1023u)];       // LDS chain
        if (OP == 9) a = __shfl_sync(0xffffffffu, a, 3);                 // broadcast shfl
        if (OP == 10) { a = a + 1.0f; }                                  // FADD
        if (OP == 11) {  // a chain of 4 uniform data-dependent branches
            const uint32_t k = __float_as_uint(a);
            if (k & 1u) a = a + 1.0f; else a = a * 0.5f;
            if (k & 2u) a = a + 3.0f; else a = a * 0.25f;
            if (k & 4u) a = a + 5.0f; else a = a * 0.125f;
            if (k & 8u) a = a + 7.0f; else a = a * 0.0625f;
        }
        if (OP == 12) {  // the same without branches (selects)
            const uint32_t k = __float_as_uint(a);
            a = (k & 1u) ? a + 1.0f : a * 0.5f;
            a = (k & 2u) ? a + 3.0f : a * 0.25f;
            a = (k & 4u) ? a + 5.0f : a * 0.125f;
            a = (k & 8u) ? a + 7.0f : a * 0.0625f;
        }
    }
    long long t1 = clock64();
    out[lane] = a + (float)u;
    if (lane == 0) cyc[0] = t1 - t0;
}

template <int OP>
static void run(const char *name, float *in, float *out, long long *cyc)
{
    const int iters = 4096;
    long long c;
    for (int r = 0; r < 2; r++) k_prim<OP><<<1, 32>>>(in, out, iters, cyc);
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-18s %6.1f cycles\n", name, (double)c / iters);
}

int main()
{
    if (ensure_fixed_tables()) return 1;
    float h[64];
    for (int i = 0; i < 64; i++) h[i] = (float)((i * 37) % 2000 - 700);
    float *in, *out;
    long long *cyc;
    cudaMalloc(&in, 256);
    cudaMalloc(&out, 256);
    cudaMalloc(&cyc, 8);
    cudaMemcpy(in, h, 256, cudaMemcpyHostToDevice);
    run<0>("fixed f", in, out, cyc);
    run<1>("shfl.idx", in, out, cyc);
    run<2>("shfl.down", in, out, cyc);
    run<3>("ballot", in, out, cyc);
    run<4>("vote.all", in, out, cyc);
    run<5>("redux.min", in, out, cyc);
    run<6>("qadd", in, out, cyc);
    run<7>("g fixed", in, out, cyc);
    run<8>("LDS chain", in, out, cyc);
    run<9>("shfl bcast", in, out, cyc);
    run<10>("fadd", in, out, cyc);
    run<11>("4 branches", in, out, cyc);
    run<12>("4 selects", in, out, cyc);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
