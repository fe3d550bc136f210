// Latency probes on the B200 (development tool): dependent-chain cycles of
// fp64 ops, global loads (L2 hit), 64-bit atomicMin, 128-bit atomicCAS.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_fp(double *out, long long *cyc, double x0, int n) {
    double x = x0, y = x0 * 0.5;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, 1.0000001, 1e-9);
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) x = sqrt(x + 1.0);
    long long t2 = clock64();
    for (int i = 0; i < n; ++i) x = 1.0 / (x + 0.5);
    long long t3 = clock64();
    for (int i = 0; i < n; ++i) x = atan2(x, y + 1.0);
    long long t4 = clock64();
    for (int i = 0; i < n; ++i) { double s, c; sincos(x, &s, &c); x = s + c * 1e-3; }
    long long t5 = clock64();
    for (int i = 0; i < n; ++i) x = x * 1.0000001 + 1e-9;  // dmul+dadd (maybe contracted)
    long long t6 = clock64();
    out[0] = x;
    cyc[0] = (t1 - t0) / n; cyc[1] = (t2 - t1) / n; cyc[2] = (t3 - t2) / n;
    cyc[3] = (t4 - t3) / n; cyc[4] = (t5 - t4) / n; cyc[5] = (t6 - t5) / n;
}

__global__ void k_fp2(double *out, long long *cyc, double x0, int n) {
    double x = x0;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = x * 1.0000001;  // dmul
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) x = x + 1e-9;  // dadd
    long long t2 = clock64();
    for (int i = 0; i < n; ++i) x = (x > 0.5 ? x : x + 1.0) * 0.999;  // dsetp + fsel + dmul
    long long t3 = clock64();
    for (int i = 0; i < n; ++i) {
        double r;
        asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
        x = r + 1e-3;
    }  // mufu rcp64h + dadd
    long long t4 = clock64();
    out[1] = x;
    cyc[8] = (t1 - t0) / n; cyc[9] = (t2 - t1) / n; cyc[10] = (t3 - t2) / n; cyc[11] = (t4 - t3) / n;
}

__global__ void k_chase(const int *next, long long *cyc, int *sink, int n, int start) {
    int j = start;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) j = __ldcg(next + j);
    long long t1 = clock64();
    sink[0] = j;
    cyc[0] = (t1 - t0) / n;
}

__global__ void k_atom(unsigned long long *a, ulonglong2 *b, long long *cyc, int n) {
    unsigned long long v = 1000000;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) v = atomicMin(a + (v & 1023), v - 1) + 0 * v + (v & 1);
    long long t1 = clock64();
    ulonglong2 c = make_ulonglong2(0, 0);
    for (int i = 0; i < n; ++i) c = atomicCAS(b + (c.x & 1023), c, make_ulonglong2(c.x + 1, c.y));
    long long t2 = clock64();
    cyc[0] = (t1 - t0) / n; cyc[1] = (t2 - t1) / n;
    a[0] = v + c.x;
}

int main() {
    double *out; long long *cyc; int *next, *sink;
    cudaMalloc(&out, 64); cudaMalloc(&cyc, 64 * 8); cudaMalloc(&sink, 64);
    k_fp<<<1, 1>>>(out, cyc, 0.7, 1000);
    long long h[8];
    cudaMemcpy(h, cyc, 64, cudaMemcpyDeviceToHost);
    printf("dfma %lld  sqrt %lld  rcp-div %lld  atan2 %lld  sincos %lld  mul+add %lld cycles\n", h[0], h[1], h[2], h[3], h[4], h[5]);
    k_fp2<<<1, 1>>>(out, cyc, 0.7, 1000);
    long long h2[16];
    cudaMemcpy(h2, cyc, 128, cudaMemcpyDeviceToHost);
    printf("dmul %lld  dadd %lld  dsetp+fsel+dmul %lld  rcp.approx+dadd %lld cycles\n", h2[8], h2[9], h2[10], h2[11]);
    // pointer chase: small (L1/L2) and large (HBM) footprints
    for (long long elems : {1LL << 10, 1LL << 20, 1LL << 24, 1LL << 27}) {
        int *hn = new int[elems];
        // random cycle with stride to defeat prefetch
        long long stride = 1; while (stride * stride < elems) stride <<= 1; stride += 1;
        for (long long i = 0; i < elems; ++i) hn[i] = (int)((i * 7919 + 104729) % elems);
        cudaMalloc(&next, elems * 4); cudaMemcpy(next, hn, elems * 4, cudaMemcpyHostToDevice);
        k_chase<<<1, 1>>>(next, cyc, sink, 2000, 1);
        k_chase<<<1, 1>>>(next, cyc, sink, 2000, 3);
        cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("chase %lld MB: %lld cycles/load\n", elems * 4 >> 20, h[0]);
        cudaFree(next); delete[] hn;
    }
    unsigned long long *a; ulonglong2 *b;
    cudaMalloc(&a, 1024 * 8); cudaMalloc(&b, 1024 * 16);
    cudaMemset(a, 0xff, 1024 * 8); cudaMemset(b, 0, 1024 * 16);
    k_atom<<<1, 1>>>(a, b, cyc, 1000);
    cudaMemcpy(h, cyc, 16, cudaMemcpyDeviceToHost);
    printf("atomicMin64 %lld  atomicCAS128 %lld cycles\n", h[0], h[1]);
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
}
