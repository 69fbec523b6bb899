// Microbenchmark: latency and throughput of the f-function variants on sm_100a.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o f_latency f_latency.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>
#define LN2_HI 0.693145751953125f
#define LN2_LO 1.42860682030941723212e-6f
#define INV_LN2 1.44269504088896341f
__device__ __forceinline__ void pq_expm(float x, float &e, float &m) {
    x = x > 100.0f ? 100.0f : x;
    const float kf = rintf(x * INV_LN2);
    float r = fmaf(-kf, LN2_HI, x); r = fmaf(-kf, LN2_LO, r);
    const float t = -r;
    float h = fmaf(t, 1.0f / 40320.0f, 1.0f / 5040.0f);
    h = fmaf(t, h, 1.0f / 720.0f); h = fmaf(t, h, 1.0f / 120.0f); h = fmaf(t, h, 1.0f / 24.0f);
    h = fmaf(t, h, 1.0f / 6.0f); h = fmaf(t, h, 0.5f);
    const float p = fmaf(t * t, h, t);
    const int k = (int)kf;
    if (k > 125) { e = 0.0f; m = 1.0f; } else {
        const float s = __uint_as_float((uint32_t)(127 - k) << 23);
        e = fmaf(s, p, s); m = fmaf(-s, p, 1.0f - s); }
}
__device__ __forceinline__ float pq_log1p_ratio(float num, float den) {
    float s, kf;
    if (num >= -0.29289322f * den && num <= 0.41421356f * den) { s = num / (2.0f * den + num); kf = 0.0f; }
    else { const float u = 1.0f + num / den; const uint32_t b = __float_as_uint(u);
        int k = (int)((b >> 23) & 0xffu) - 127; float mm = __uint_as_float((b & 0x007fffffu) | 0x3f800000u);
        if (mm > 1.41421356f) { mm *= 0.5f; k += 1; } s = (mm - 1.0f) / (mm + 1.0f); kf = (float)k; }
    const float z = s * s;
    float h = fmaf(z, 1.0f / 11.0f, 1.0f / 9.0f); h = fmaf(z, h, 1.0f / 7.0f); h = fmaf(z, h, 1.0f / 5.0f);
    h = fmaf(z, h, 1.0f / 3.0f);
    const float s2 = s + s; const float p = fmaf(s2 * z, h, s2);
    return fmaf(kf, LN2_HI, fmaf(kf, LN2_LO, p));
}
__device__ __forceinline__ float fmag_exact(float a, float b) {
    const float lo = fminf(a, b), hi = fmaxf(a, b); const bool big = lo > 40.0f;
    float e1, m1, e2, m2; pq_expm(big ? hi - lo : lo, e1, m1); pq_expm(hi, e2, m2);
    const float num = big ? -e1 : m1 * m2; const float den = big ? 1.0f + e1 : e1 + e2;
    const float base = big ? lo : 0.0f; return base + pq_log1p_ratio(num, den);
}
// MUFU-based (not reproducible on CPU): |f| = min + log1p(e^-(a+b)) - log1p(e^-|a-b|)
// for lo >= 1, tanh form for small
__device__ __forceinline__ float fmag_mufu(float a, float b) {
    const float lo = fminf(a, b), hi = fmaxf(a, b);
    float e1 = exp2f(-(hi + lo) * 1.44269504f), e2 = exp2f(-(hi - lo) * 1.44269504f);
    return lo + (log2f(1.0f + e1) - log2f(1.0f + e2)) * 0.69314718f;
}
template <int MODE>
__global__ void lat(const float *in, float *out, int iters, long long *cyc) {
    float a = in[threadIdx.x], b = in[threadIdx.x + 32];
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        float r;
        if (MODE == 0) r = fmag_exact(a, b); else if (MODE == 1) r = fmag_mufu(a, b); else r = fminf(a, b);
        a = r + 0.5f;  // keep magnitudes in range, dependent chain
        b = b * 1.0001f;
    }
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
template <int MODE, int ILP>
__global__ void thr(const float *in, float *out, int iters) {
    float a[ILP], b = in[threadIdx.x];
    for (int k = 0; k < ILP; k++) a[k] = in[(threadIdx.x + k) & 63] + k;
    for (int i = 0; i < iters; i++)
        for (int k = 0; k < ILP; k++) {
            float r = MODE == 0 ? fmag_exact(a[k], b) : (MODE == 1 ? fmag_mufu(a[k], b) : fminf(a[k], b));
            a[k] = r + 0.5f;
        }
    float s = 0; for (int k = 0; k < ILP; k++) s += a[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    float h[64]; for (int i = 0; i < 64; i++) h[i] = 0.3f + 0.37f * i;
    float *in, *out; long long *cyc; cudaMalloc(&in, 256); cudaMalloc(&out, 1 << 26); cudaMalloc(&cyc, 8);
    cudaMemcpy(in, h, 256, cudaMemcpyHostToDevice);
    const int iters = 4096; long long c;
    const char *names[] = {"exact-ieee", "mufu", "minsum"};
    for (int m = 0; m < 3; m++) {
        for (int rep = 0; rep < 2; rep++) {
            if (m == 0) lat<0><<<1, 32>>>(in, out, iters, cyc); else if (m == 1) lat<1><<<1, 32>>>(in, out, iters, cyc); else lat<2><<<1, 32>>>(in, out, iters, cyc);
            cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        }
        printf("%-11s latency per f (incl +0.5 add): %.1f cycles\n", names[m], (double)c / iters);
    }
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int m = 0; m < 3; m++) {
        for (int rep = 0; rep < 2; rep++) {
            cudaEventRecord(e0);
            if (m == 0) thr<0, 8><<<sms * 8, 256>>>(in, out, 256); else if (m == 1) thr<1, 8><<<sms * 8, 256>>>(in, out, 256); else thr<2, 8><<<sms * 8, 256>>>(in, out, 256);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
        }
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double nf = (double)sms * 8 * 256 * 256 * 8;
        printf("%-11s throughput: %.3g f/s (%.2f ms)\n", names[m], nf / (ms * 1e-3), ms);
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
