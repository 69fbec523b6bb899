// Dependent-chain latencies of the serial engine's primitives (cycles per op).
#include <cstdio>
#include "../../paper_1204_5882_b200/csrc/polarsc.cu"
#include "../../paper_1204_5882_b200/csrc/serial_q88.cuh"
#define N 2000
template <int K>
__global__ void kp(const int *in, long long *cyc, int *out)
{
    se::load_tables();
    for (int i = threadIdx.x; i < CORR_SMEM; i += blockDim.x) pq_corrtab[i] = CORR_TAB_C[i];
    __syncwarp();
    int a = in[threadIdx.x], b = in[threadIdx.x + 32];
    long long t0 = clock64();
#pragma unroll 4
    for (int r = 0; r < N; r++) {
        if (K == 0) a = se::fq(a, b);
        if (K == 1) a = se::qa(a, b);
        if (K == 2) a = se::ctab[a & 2047] + b;
        if (K == 3) a = __shfl_sync(0xffffffffu, a, b & 31);
        if (K == 4) a = __shfl_down_sync(0xffffffffu, a, 8);
        if (K == 5) a = (int)__ballot_sync(0xffffffffu, a < b);
        if (K == 6) a = __all_sync(0xffffffffu, a < b) ? a + 1 : a - 1;
        if (K == 7) a = __reduce_add_sync(0xffffffffu, a) & 1023;
        if (K == 8) a = (a < b) ? a + 3 : b - a;
        if (K == 9) a = __float_as_int(pq_f<PQ_F_FIXED>(__int_as_float(a), __int_as_float(b)));
        if (K == 10) a = se::gq(a, b, a & 1);
        if (K == 11) { if (a & 1) a = a * 3 + 1; else a = a >> 1; }
        if (K == 12) a = __shfl_sync(0xffffffffu, a, 0);
    }
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) / N;
}
template <int K>
void run(const char *nm, const int *din, long long *dc, int *dout)
{
    long long c;
    kp<K><<<1, 32>>>(din, dc, dout);
    kp<K><<<1, 32>>>(din, dc, dout);
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    printf("%-28s %4lld cycles\n", nm, c);
}
int main()
{
    ensure_fixed_tables();
    int h[64];
    for (int i = 0; i < 64; i++) h[i] = (i * 7919) % 3000 - 1500;
    int *din, *dout; long long *dc;
    cudaMalloc(&din, 256); cudaMalloc(&dout, 256); cudaMalloc(&dc, 8);
    cudaMemcpy(din, h, 256, cudaMemcpyHostToDevice);
    run<0>("int fq (table boxplus)", din, dc, dout);
    run<9>("float pq_f fixed", din, dc, dout);
    run<1>("qa (sat add)", din, dc, dout);
    run<10>("gq", din, dc, dout);
    run<2>("LDS.U8 + IADD", din, dc, dout);
    run<3>("shfl.idx (lane var)", din, dc, dout);
    run<12>("shfl.idx (const 0)", din, dc, dout);
    run<4>("shfl.down 8", din, dc, dout);
    run<5>("ballot", din, dc, dout);
    run<6>("vote.all + sel", din, dc, dout);
    run<7>("redux.add", din, dc, dout);
    run<8>("isetp + sel/add", din, dc, dout);
    run<11>("branchy collatz", din, dc, dout);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
