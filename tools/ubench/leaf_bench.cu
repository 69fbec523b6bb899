// Width-32 engine microbenchmark on a config's real sub-tree sequence
// (tools/ubench/gen_leaf_types.py): one warp per CTA, cycles per sub-tree,
// fixed-point f.  Includes the product source.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 -I../../include -o leaf_bench leaf_bench.cu
#include <cstdio>
#include <cstring>
#include <vector>
#ifndef NO_UB
#define PQ_UBENCH_TIMING 1
#endif
#include "../../paper_1204_5882_b200/csrc/polarsc.cu"

__device__ __forceinline__ uint32_t hash32(uint32_t x)
{
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}

__device__ __forceinline__ float qval(uint32_t i, int lane, int spread)
{
    const uint32_t h = hash32(i * 32u + (uint32_t)lane);
    // Q8.8 code: mostly reliable positive values, a few weak / negative ones
    const int mag = (int)(h & 4095u) + (int)((h >> 12) & 1023u) * spread;
    return (float)(((h >> 30) == 0u) ? -mag : mag);
}

template <int FM, int ENG>
__global__ void k_leaf(const TypeBits *T, int n, int reps, int spread, long long *cyc, uint32_t *out, int sel = -1)
{
    load_log_table();
    for (int i = threadIdx.x; i < 4097; i += blockDim.x) pq_corrtab[i] = CORR_TAB_C[i];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    NodePos np;
    np.dump = nullptr; np.N = 32; np.d = 0; np.j = 0;
    uint32_t acc = 0;
    long long t0 = clock64();
    for (int r = 0; r < reps; r++)
        for (int i = 0; i < n; i++) {
            const TypeBits t = T[sel >= 0 ? sel : i];
            const float v = qval((uint32_t)i + 977u * r, lane, spread) + (float)(acc & 1u);
            uint32_t b;
            b = dec32<FM, false>(v, t, np);
            acc = acc * 3u + b;
        }
    long long t1 = clock64();
    out[blockIdx.x * 32 + lane] = acc;
    if (lane == 0 && blockIdx.x == 0) cyc[0] = (t1 - t0) / ((long long)reps * n);
}

// the whole single-warp band on width-512 sub-trees: types staged to shared
// memory, node values filled, then the product's warp_walk (timed alone)
template <int FM, int V2>
__global__ void k_walk(const uint8_t *ty_g, int n, int spread, long long *cyc, uint32_t *out, uint32_t *bits)
{
    __shared__ __align__(16) uint8_t ty[1024];
    __shared__ __align__(16) float st[1024];
    __shared__ uint32_t xs[16];
    load_log_table();
    for (int i = threadIdx.x; i < 4097; i += blockDim.x) pq_corrtab[i] = CORR_TAB_C[i];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    long long tot = 0;
    uint32_t acc = 0;
    for (int i = 0; i < n; i++) {
        for (int q = lane; q < 64; q += 32)
            reinterpret_cast<uint4 *>(ty)[q] = reinterpret_cast<const uint4 *>(ty_g + 1024 * (size_t)i)[q];
        for (int q = 0; q < 16; q++) st[32 * q + lane] = qval((uint32_t)(16 * i + q), lane, spread);
        __syncwarp();
        const long long t0 = clock64();
        if (V2) warp_walk2<FM>(st + 1024, xs, ty, 512, 0, 0, 0);
        else warp_walk<FM>(st + 1024, xs, ty, nullptr, 512, 512, 0, 0, 0, 0, 0);
        acc = acc * 3u + xs[lane & 15];
        tot += clock64() - t0;
        __syncwarp();
        if (blockIdx.x == 0 && lane < 16) bits[16 * i + lane] = xs[lane];
    }
    out[blockIdx.x * 32 + lane] = acc;
    if (lane == 0 && blockIdx.x == 0) cyc[0] = tot / n;
}

static void ub_report(const char *tag)
{
#ifdef NO_UB
    return;
#else
    unsigned long long t[16], n[16], z[16] = {0};
    cudaMemcpyFromSymbol(t, g_ub_time, sizeof t);
    cudaMemcpyFromSymbol(n, g_ub_count, sizeof n);
    cudaMemcpyToSymbol(g_ub_time, z, sizeof z);
    cudaMemcpyToSymbol(g_ub_count, z, sizeof z);
    const char *nm[7] = {"dec8gen", "dec32", "walk", "dec16gen", "dec8pat", "dec8spec", "dec16spec"};
    printf("   %s:", tag);
    for (int i = 0; i < 7; i++)
        if (n[i]) printf(" %s %.0fx%.0f", nm[i], (double)n[i], (double)t[i] / n[i]);
    printf("\n");
#endif
}

static TypeBits make_tb(const uint8_t *t)
{
    TypeBits T{0, 0, 0};
    for (int h = 1; h < 32; h++) {
        T.tb0 |= (uint32_t)(t[h] & 1u) << h;
        T.tb1 |= (uint32_t)((t[h] >> 1) & 1u) << h;
    }
    for (int h = 32; h < 64; h++) T.leaf |= (uint32_t)(t[h] == NT_RATE0) << (h - 32);
    return T;
}

int main(int argc, char **argv)
{
    const char *path = argc > 1 ? argv[1] : "leaf_c3.bin";
    FILE *f = fopen(path, "rb");
    if (!f) { printf("no %s\n", path); return 1; }
    std::vector<uint8_t> raw;
    uint8_t buf[64];
    while (fread(buf, 1, 64, f) == 64) raw.insert(raw.end(), buf, buf + 64);
    fclose(f);
    const int n = (int)(raw.size() / 64);
    std::vector<TypeBits> tb(n);
    for (int i = 0; i < n; i++) tb[i] = make_tb(&raw[64 * i]);
    // fixed tables (RATE1_TAU_FIX, CORR_TAB_C) as the library sets them up
    if (ensure_fixed_tables()) { printf("tables: %s\n", pq_last_error()); return 1; }
    TypeBits *d_tb; long long *d_cyc; uint32_t *d_out;
    cudaMalloc(&d_tb, n * sizeof(TypeBits));
    cudaMalloc(&d_cyc, 8);
    cudaMalloc(&d_out, 148 * 32 * 4);
    cudaMemcpy(d_tb, tb.data(), n * sizeof(TypeBits), cudaMemcpyHostToDevice);
    long long c;
    for (int grid : {1, 148})
        for (int spread : {0, 4}) {
            uint32_t o0[32];
            for (int r = 0; r < 2; r++) k_leaf<PQ_F_FIXED, 0><<<grid, 32>>>(d_tb, n, 2, spread, d_cyc, d_out);
            cudaMemcpy(&c, d_cyc, 8, cudaMemcpyDeviceToHost);
            cudaMemcpy(o0, d_out, 128, cudaMemcpyDeviceToHost);
            printf("product dec32 fixed  grid %3d spread %d: %lld cycles per width-32 sub-tree (%d sub-trees)\n",
                   grid, spread, c, n);

        }
    // single patterns repeated (warm instruction cache, one path)
    {
        int shown = 0;
        for (int i = 0; i < n && shown < 10; i++) {
            if (((tb[i].tb0 >> 1) & 1u) || ((tb[i].tb1 >> 1) & 1u)) continue;  // mixed roots only
            if (i % 97) continue;
            shown++;
            long long c0;
            for (int r = 0; r < 2; r++) k_leaf<PQ_F_FIXED, 0><<<1, 32>>>(d_tb, n, 1, 4, d_cyc, d_out, i);
            cudaMemcpy(&c0, d_cyc, 8, cudaMemcpyDeviceToHost);
            printf("pattern %4d tb0 %08x tb1 %08x leaf %08x: dec32 %lld cycles (repeated, warm)\n", i, tb[i].tb0,
                   tb[i].tb1, tb[i].leaf, c0);
        }
    }
    const char *p512 = argc > 2 ? argv[2] : "w512_c3.bin";
    if ((f = fopen(p512, "rb"))) {
        std::vector<uint8_t> r5;
        uint8_t b5[1024];
        while (fread(b5, 1, 1024, f) == 1024) r5.insert(r5.end(), b5, b5 + 1024);
        fclose(f);
        const int n5 = (int)(r5.size() / 1024);
        uint8_t *d_ty;
        uint32_t *d_b0, *d_b1;
        cudaMalloc(&d_b0, n5 * 64);
        cudaMalloc(&d_b1, n5 * 64);
        cudaMalloc(&d_ty, r5.size());
        cudaMemcpy(d_ty, r5.data(), r5.size(), cudaMemcpyHostToDevice);
        for (int grid : {1, 148})
            for (int spread : {0, 4}) {
                k_walk<PQ_F_FIXED, 0><<<grid, 32>>>(d_ty, n5, spread, d_cyc, d_out, d_b0);
                cudaDeviceSynchronize();
                ub_report("warm");
                k_walk<PQ_F_FIXED, 0><<<grid, 32>>>(d_ty, n5, spread, d_cyc, d_out, d_b0);
                cudaDeviceSynchronize();
                if (grid == 1) ub_report("walk ");
                cudaMemcpy(&c, d_cyc, 8, cudaMemcpyDeviceToHost);
                printf("product warp_walk  fixed grid %3d spread %d: %lld cycles per width-512 sub-tree (%d)\n",
                       grid, spread, c, n5);
                k_walk<PQ_F_FIXED, 1><<<grid, 32>>>(d_ty, n5, spread, d_cyc, d_out, d_b1);
                cudaDeviceSynchronize();
                ub_report("warm");
                k_walk<PQ_F_FIXED, 1><<<grid, 32>>>(d_ty, n5, spread, d_cyc, d_out, d_b1);
                cudaDeviceSynchronize();
                if (grid == 1) ub_report("walk2");
                cudaMemcpy(&c, d_cyc, 8, cudaMemcpyDeviceToHost);
                std::vector<uint32_t> h0(n5 * 16), h1(n5 * 16);
                cudaMemcpy(h0.data(), d_b0, n5 * 64, cudaMemcpyDeviceToHost);
                cudaMemcpy(h1.data(), d_b1, n5 * 64, cudaMemcpyDeviceToHost);
                int bad = 0;
                for (int q = 0; q < n5 * 16; q++) bad += h0[q] != h1[q];
                printf("         warp_walk2 fixed grid %3d spread %d: %lld cycles per width-512 sub-tree; %d words differ\n",
                       grid, spread, c, bad);
            }
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
