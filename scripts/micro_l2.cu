// Micro-benchmark: the L2 -> SM read bandwidth of B200 for L2-resident data
// (the ceiling of the gather traffic of the filter SpMM), and HBM streaming
// read / copy for reference.  16-byte and 32-byte loads, L1 bypassed (.cg).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/micro_l2.cu -o micro_l2
#include <cuda_runtime.h>
#include <stdio.h>

__global__ void read_cg16(const double2 *__restrict__ p, size_t n, int reps, double *out) {
    double2 acc = make_double2(0, 0);
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
            double2 v = __ldcg(p + i);
            acc.x += v.x;
            acc.y += v.y;
        }
    if (acc.x == 1234.5) out[0] = acc.y;
}

__global__ void read_cg32(const double *__restrict__ p, size_t n4, int reps, double *out) {
    double a = 0;
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
            double x0, x1, x2, x3;
            asm volatile("ld.global.cg.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(x0), "=d"(x1), "=d"(x2), "=d"(x3)
                         : "l"(p + 4 * i));
            a += x0 + x1 + x2 + x3;
        }
    if (a == 1234.5) out[0] = a;
}

__global__ void copy16(const double2 *__restrict__ s, double2 *__restrict__ d, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        __stcs(d + i, __ldcs(s + i));
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *out;
    cudaMalloc(&out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto t = [&](const char *name, double bytes, auto fn) {
        fn();
        cudaDeviceSynchronize();
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0);
            fn();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
        }
        printf("%-48s %8.3f ms  %8.1f GB/s\n", name, best, bytes / best / 1e6);
    };
    for (size_t mb : {16, 32, 64, 96}) {
        size_t bytes = mb << 20;
        double *buf;
        cudaMalloc(&buf, bytes);
        cudaMemset(buf, 0, bytes);
        int reps = (int)(4096 / mb);
        for (int tpb : {256, 512}) {
            for (int bps : {2, 4}) {
                char nm[128];
                snprintf(nm, sizeof nm, "L2 read16 %zuMB tpb=%d ctas/sm=%d", mb, tpb, bps);
                t(nm, (double)bytes * reps, [&] { read_cg16<<<sms * bps, tpb>>>((double2 *)buf, bytes / 16, reps, out); });
                snprintf(nm, sizeof nm, "L2 read32 %zuMB tpb=%d ctas/sm=%d", mb, tpb, bps);
                t(nm, (double)bytes * reps, [&] { read_cg32<<<sms * bps, tpb>>>(buf, bytes / 32, reps, out); });
            }
        }
        cudaFree(buf);
    }
    size_t big = (size_t)4 << 30;
    double *a, *b;
    cudaMalloc(&a, big);
    cudaMalloc(&b, big);
    cudaMemset(a, 0, big);
    t("HBM read16 4GB", (double)big, [&] { read_cg16<<<sms * 4, 512>>>((double2 *)a, big / 16, 1, out); });
    t("HBM read32 4GB", (double)big, [&] { read_cg32<<<sms * 4, 512>>>(a, big / 32, 1, out); });
    t("HBM copy16 4GB (r+w bytes)", 2.0 * big, [&] { copy16<<<sms * 4, 512>>>((double2 *)a, (double2 *)b, big / 16); });
    return 0;
}
