// DMMA.8x8x4 issue-rate ceiling on this GPU: independent accumulators in registers,
// no memory traffic in the loop. Reports TFLOP/s for several warps-per-SM settings.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
template <int NACC>
__global__ void k(double *out, int iters) {
    double acc[NACC][2];
    double a = threadIdx.x * 1e-3, b = blockIdx.x * 1e-3;
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i][0] = acc[i][1] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NACC; ++i) dmma(acc[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1];
    if (s == 1.2345) out[0] = s;
}
template <int NACC>
void run(int threads, int ctas_per_sm, int sms) {
    double *o;
    cudaMalloc(&o, 8);
    const int iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<NACC><<<sms * ctas_per_sm, threads>>>(o, 16);
    cudaEventRecord(e0);
    k<NACC><<<sms * ctas_per_sm, threads>>>(o, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 512.0 * NACC * iters * (threads / 32) * (double)sms * ctas_per_sm;
    printf("NACC=%2d threads=%4d ctas/sm=%d  %.2f TFLOP/s\n", NACC, threads, ctas_per_sm, flops / ms / 1e9);
    cudaFree(o);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int t : {128, 256, 512}) for (int c : {1, 2, 4}) { run<8>(t, c, sms); run<16>(t, c, sms); }
    return 0;
}
