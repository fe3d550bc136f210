// Accuracy of MUFU-seeded fp64 division / square root sequences against
// IEEE (development tool): counts results differing from a / b and
// sqrt(x) over random operands spanning many binades.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double div2(double a, double b) {  // two Newton steps (current)
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b));
    double e = fma(-b, r, 1.0);
    r = fma(r, e, r);
    e = fma(-b, r, 1.0);
    r = fma(r, e, r);
    const double q = a * r;
    return fma(fma(-b, q, a), r, q);
}
__device__ __forceinline__ double div3(double a, double b) {  // one cubic step
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b));
    double e = fma(-b, r, 1.0);
    e = fma(e, e, e);
    r = fma(r, e, r);
    const double q = a * r;
    return fma(fma(-b, q, a), r, q);
}
__device__ __forceinline__ double sq2(double x) {  // current
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double h = 0.5 * x;
    y = y * fma(-h * y, y, 1.5);
    y = y * fma(-h * y, y, 1.5);
    const double s = x * y;
    const double r = fma(fma(-s, s, x), 0.5 * y, s);
    return x > 0.0 ? r : 0.0;
}
__device__ __forceinline__ double sq3(double x) {  // one cubic step
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double e = fma(-x * y, y, 1.0);             // 1 - x y^2
    y = fma(y * e, fma(e, 0.375, 0.5), y);            // y (1 + e/2 + 3e^2/8)
    const double s = x * y;
    const double r = fma(fma(-s, s, x), 0.5 * y, s);
    return x > 0.0 ? r : 0.0;
}

__device__ unsigned long long mix(unsigned long long z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__device__ double rnd(unsigned long long s) {  // mantissa random, exponent in [-40, 40]
    const unsigned long long m = mix(s);
    const double f = 1.0 + (double)(m >> 12) * 0x1p-52;
    const int e = (int)((mix(s ^ 0x1234) % 81)) - 40;
    return ldexp(f, e);
}

__global__ void k(unsigned long long *cnt, long long n) {
    unsigned long long c[6] = {0, 0, 0, 0, 0, 0};
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double a = rnd(2 * i), b = rnd(2 * i + 1);
        const double q = a / b, s = sqrt(a);
        const double q2 = div2(a, b), q3 = div3(a, b), s2 = sq2(a), s3 = sq3(a);
        c[0] += q2 != q;
        c[1] += q3 != q;
        c[2] += s2 != s;
        c[3] += s3 != s;
        const long long d3 = __double_as_longlong(q3) - __double_as_longlong(q);
        const long long e3 = __double_as_longlong(s3) - __double_as_longlong(s);
        c[4] += (d3 > 1 || d3 < -1);
        c[5] += (e3 > 1 || e3 < -1);
    }
    for (int j = 0; j < 6; ++j) atomicAdd(cnt + j, c[j]);
}

int main() {
    unsigned long long *d, h[6];
    cudaMalloc(&d, 48);
    cudaMemset(d, 0, 48);
    const long long n = 1LL << 28;
    k<<<148 * 8, 256>>>(d, n);
    cudaMemcpy(h, d, 48, cudaMemcpyDeviceToHost);
    printf("n=%lld  div2!=ieee %llu  div3!=ieee %llu  sqrt2!=ieee %llu  sqrt3!=ieee %llu  div3>1ulp %llu  sqrt3>1ulp %llu\n",
           n, h[0], h[1], h[2], h[3], h[4], h[5]);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
