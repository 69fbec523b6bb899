#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
// dispatch cost: switch over dense ids (jump table) vs compare chain, one warp, dependent chain
template <int K> __device__ __forceinline__ int body(int x) {
    // distinct small straight-line work per case (so cases do not merge)
    #pragma unroll
    for (int i = 0; i < 3; i++) x = (x ^ (K * 2654435761u + i)) + (x >> (K + 1));
    return x;
}
__global__ void k_switch(const uint8_t *ids, int n, int reps, int *out, long long *cyc) {
    __shared__ uint8_t s[4096];
    for (int i = threadIdx.x; i < n; i += 32) s[i] = ids[i];
    __syncwarp();
    int x = threadIdx.x;
    long long t0 = clock64();
    for (int r = 0; r < reps; r++)
        for (int i = 0; i < n; i++) {
            switch (s[i]) {
            case 0: x = body<0>(x); break; case 1: x = body<1>(x); break; case 2: x = body<2>(x); break;
            case 3: x = body<3>(x); break; case 4: x = body<4>(x); break; case 5: x = body<5>(x); break;
            case 6: x = body<6>(x); break; case 7: x = body<7>(x); break; case 8: x = body<8>(x); break;
            case 9: x = body<9>(x); break; case 10: x = body<10>(x); break; case 11: x = body<11>(x); break;
            case 12: x = body<12>(x); break; case 13: x = body<13>(x); break; case 14: x = body<14>(x); break;
            default: x = body<15>(x); break;
            }
        }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_chain(const uint8_t *ids, int n, int reps, int *out, long long *cyc) {
    __shared__ uint8_t s[4096];
    for (int i = threadIdx.x; i < n; i += 32) s[i] = ids[i];
    __syncwarp();
    int x = threadIdx.x;
    long long t0 = clock64();
    for (int r = 0; r < reps; r++)
        for (int i = 0; i < n; i++) {
            const int id = s[i];
            if (id == 0) x = body<0>(x); else if (id == 1) x = body<1>(x); else if (id == 2) x = body<2>(x);
            else if (id == 3) x = body<3>(x); else if (id == 4) x = body<4>(x); else if (id == 5) x = body<5>(x);
            else if (id == 6) x = body<6>(x); else if (id == 7) x = body<7>(x); else if (id == 8) x = body<8>(x);
            else if (id == 9) x = body<9>(x); else if (id == 10) x = body<10>(x); else if (id == 11) x = body<11>(x);
            else if (id == 12) x = body<12>(x); else if (id == 13) x = body<13>(x); else if (id == 14) x = body<14>(x);
            else x = body<15>(x);
        }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_none(const uint8_t *ids, int n, int reps, int *out, long long *cyc) {
    __shared__ uint8_t s[4096];
    for (int i = threadIdx.x; i < n; i += 32) s[i] = ids[i];
    __syncwarp();
    int x = threadIdx.x;
    long long t0 = clock64();
    for (int r = 0; r < reps; r++)
        for (int i = 0; i < n; i++) x = body<3>(x) + s[i];
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    const int n = 4096, reps = 20;
    uint8_t h[n]; uint32_t r = 12345;
    uint8_t *d; int *o; long long *c, hc;
    cudaMalloc(&d, n); cudaMalloc(&o, 128); cudaMalloc(&c, 8);
    for (int mode = 0; mode < 3; mode++) {
        for (int i = 0; i < n; i++) { r = r * 1664525u + 1013904223u; h[i] = mode == 0 ? (r >> 24) & 15 : mode == 1 ? (r >> 24) & 3 : 5; }
        cudaMemcpy(d, h, n, cudaMemcpyHostToDevice);
        for (int w = 0; w < 2; w++) {
        k_switch<<<1, 32>>>(d, n, reps, o, c); cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
        printf("mode %d switch: %.1f cycles/iter\n", mode, (double)hc / (n * reps));
        k_chain<<<1, 32>>>(d, n, reps, o, c); cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
        printf("mode %d chain : %.1f cycles/iter\n", mode, (double)hc / (n * reps));
        k_none<<<1, 32>>>(d, n, reps, o, c); cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
        printf("mode %d none  : %.1f cycles/iter\n", mode, (double)hc / (n * reps));
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
