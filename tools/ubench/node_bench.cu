// Latency of individual lower-band building blocks (one warp, dependent chain).
#include "../../paper_1204_5882_b200/csrc/polarsc.cu"
#ifndef FMX
#define FMX PQ_F_EXACT
#endif

template <int MODE, bool PL>
__device__ __forceinline__ uint32_t node(float v, const TypeBits &T, const NodePos &np)
{
    if (MODE == 8) return dec8<FMX, PL>(v, T, 1, np);
    if (MODE == 32) return dec32<FMX, PL>(v, T, np);
    if (MODE == 16) return dec16<FMX, PL>(v, T, 1, np);
    if (MODE == 4)
        return dec4<FMX, PL>(__shfl_sync(0xffffffffu, v, 0), __shfl_sync(0xffffffffu, v, 1), __shfl_sync(0xffffffffu, v, 2),
                             __shfl_sync(0xffffffffu, v, 3), T, 1, np);
    return dec2<FMX, PL>(v, __shfl_sync(0xffffffffu, v, 1), T, 1, np);
}

template <int MODE>
__global__ void k_node(const float *in, long long *cyc, uint32_t *out, int iters, uint32_t tb0, uint32_t tb1,
                       uint32_t leaf, int plain)
{
    load_log_table();
    __syncthreads();
    TypeBits T;
    T.tb0 = tb0;
    T.tb1 = tb1;
    T.leaf = leaf;
    NodePos np;
    np.dump = nullptr;
    np.N = 32;
    np.d = 0;
    np.j = 0;
    float v = in[threadIdx.x & 31];
    uint32_t acc = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        uint32_t r;
        if (plain) r = node<MODE, true>(v, T, np);
        else r = node<MODE, false>(v, T, np);
        acc += r;
        v = v + 1e-7f * (float)(r & 1u);  // carry a dependency into the next call
    }
    long long t1 = clock64();
    out[threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) / iters;
}

int main()
{
    float h[32];
    for (int i = 0; i < 32; i++) h[i] = (i % 3 == 0 ? -1.f : 1.f) * (2.0f + 0.37f * (i % 7));
    float *in;
    long long *cyc, c;
    uint32_t *out;
    cudaMalloc(&in, 128);
    cudaMalloc(&cyc, 8);
    cudaMalloc(&out, 128);
    cudaMemcpy(in, h, 128, cudaMemcpyHostToDevice);
    auto run = [&](const char *name, auto kern, uint32_t tb0, uint32_t tb1, uint32_t leaf, int plain) {
        for (int r = 0; r < 2; r++) kern<<<1, 32>>>(in, cyc, out, 200, tb0, tb1, leaf, plain);
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        printf("%-40s %7lld cycles\n", name, c);
    };
    // type codes: MIXED 0, R0 1, R1 2, REP 3 -> tb0 = bit0, tb1 = bit1 per heap index
    // all internal nodes R1: tb0 = 0, tb1 = all
    run("dec2 R1 (guard)", k_node<2>, 0u, 0xffffffffu, 0u, 0);
    run("dec2 REP", k_node<2>, 0xffffffffu, 0xffffffffu, 0u, 0);
    run("dec2 mixed (I,I generic)", k_node<2>, 0u, 0u, 0u, 1);
    run("dec4 R1", k_node<4>, 0u, 0xffffffffu, 0u, 0);
    run("dec4 plain (3 mixed)", k_node<4>, 0u, 0u, 0u, 1);
    run("dec8 R1", k_node<8>, 0u, 0xffffffffu, 0u, 0);
    run("dec8 plain (7 mixed)", k_node<8>, 0u, 0u, 0u, 1);
    run("dec16 plain (15 mixed)", k_node<16>, 0u, 0u, 0u, 1);
    run("dec32 R1", k_node<32>, 0u, 0xffffffffu, 0u, 0);
    run("dec32 plain (31 mixed)", k_node<32>, 0u, 0u, 0u, 1);
    // mixed root whose children are R1 (types: h=1 mixed, h>=2 R1)
    run("dec8 mixed root, R1 children", k_node<8>, 0u, 0xfffffffcu, 0u, 0);
    run("dec4 mixed root, REP+R1 children", k_node<4>, 0x4u, 0xcu, 0u, 0);
    // the launch profiled by ncu: 148 warps, dec8 mixed root with R1 children
    k_node<8><<<148, 32>>>(in, cyc, out, 2000, 0u, 0xfffffffcu, 0u, 0);
    cudaDeviceSynchronize();
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
