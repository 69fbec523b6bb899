// Width-8 node decoders in isolation: cycles per call (dependent chain of
// calls), product lane-parallel dec8 vs the replicated serial_q88 routines.
#include <cstdio>
#include "../../paper_1204_5882_b200/csrc/polarsc.cu"
#include "../../paper_1204_5882_b200/csrc/serial_q88.cuh"

__device__ __forceinline__ uint32_t hash32(uint32_t x)
{
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}
__device__ __forceinline__ int qv(uint32_t i, int lane)
{
    const uint32_t h = hash32(i * 32u + (uint32_t)lane);
    const int mag = (int)(h & 2047u) + 200;
    return ((h >> 29) == 0u) ? -mag : mag;
}

template <int ENG, uint32_t PAT>
__global__ void k8(int reps, long long *cyc, uint32_t *out)
{
    load_log_table();
    for (int i = threadIdx.x; i < CORR_SMEM; i += blockDim.x) pq_corrtab[i] = CORR_TAB_C[i];
    se::load_tables();
    __syncwarp();
    const int lane = threadIdx.x & 31;
    uint32_t acc = 0;
    TypeBits T;  // width-8 node at heap h = 4 of a width-32 TypeBits: leaf bits 0..7
    T.tb0 = 0; T.tb1 = 0; T.leaf = PAT;
    long long t0 = clock64();
    for (int r = 0; r < reps; r++) {
        const int v = qv((uint32_t)r, lane) + (int)(acc & 1u);
        uint32_t b;
        if (ENG == 0) {
            NodePos np; np.dump = nullptr; np.N = 0; np.d = 0; np.j = 0;
            b = dec8<PQ_F_FIXED, false>((float)v, T, 4, np);
        } else {
            int x[8];
#pragma unroll
            for (int i = 0; i < 8; i++) x[i] = __shfl_sync(0xffffffffu, v, i);
            b = ENG == 1 ? se::d8(x, PAT) : se::rplain<8>(x, PAT);
        }
        acc = acc * 3u + b;
    }
    long long t1 = clock64();
    out[lane] = acc;
    if (lane == 0) cyc[0] = (t1 - t0) / reps;
}

template <uint32_t PAT>
void run(long long *d_cyc, uint32_t *d_out)
{
    long long c[3];
    uint32_t o[3];
    k8<0, PAT><<<1, 32>>>(1000, d_cyc, d_out); cudaMemcpy(&c[0], d_cyc, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&o[0], d_out, 4, cudaMemcpyDeviceToHost);
    k8<1, PAT><<<1, 32>>>(1000, d_cyc, d_out); cudaMemcpy(&c[1], d_cyc, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&o[1], d_out, 4, cudaMemcpyDeviceToHost);
    k8<2, PAT><<<1, 32>>>(1000, d_cyc, d_out); cudaMemcpy(&c[2], d_cyc, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&o[2], d_out, 4, cudaMemcpyDeviceToHost);
    printf("pattern %02x: product dec8 %4lld  replicated %4lld  plain %4lld cycles/call  %s\n", PAT, c[0], c[1], c[2],
           (o[0] == o[1] && o[1] == o[2]) ? "same bits" : "BITS DIFFER");
}

int main()
{
    if (ensure_fixed_tables()) { printf("%s\n", pq_last_error()); return 1; }
    int ti[26]; float tf[26], corr[4097];
    fixed_tables(corr, tf);
    for (int k = 0; k < 26; k++) ti[k] = tf[k] > 1e9f ? 0x7fffffff : (int)tf[k];
    cudaMemcpyToSymbol(se::TAUI, ti, sizeof ti);
    long long *d_cyc; uint32_t *d_out;
    cudaMalloc(&d_cyc, 8); cudaMalloc(&d_out, 128);
    run<0x01>(d_cyc, d_out); run<0x17>(d_cyc, d_out); run<0x1F>(d_cyc, d_out); run<0x07>(d_cyc, d_out);
    run<0x03>(d_cyc, d_out); run<0x3F>(d_cyc, d_out); run<0x00>(d_cyc, d_out); run<0x7F>(d_cyc, d_out);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
