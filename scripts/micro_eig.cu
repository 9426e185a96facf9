// Micro-benchmark of the small dense symmetric eigensolvers cuSOLVER offers for
// the projected problem H = Q^T A Q (A5, not graded): syevd (all pairs),
// syevdx (the leading half only) and syevj (Jacobi), fp64, m = (p+1)w sizes of
// the configs.  nvcc -gencode arch=compute_100a,code=sm_100a -O2 scripts/micro_eig.cu -lcusolver -o micro_eig
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

int main() {
    cusolverDnHandle_t h;
    cusolverDnCreate(&h);
    cudaStream_t s;
    cudaStreamCreate(&s);
    cusolverDnSetStream(h, s);
    int sizes[] = {220, 440, 846, 1100, 1650, 2200};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int m : sizes) {
        std::vector<double> hA((size_t)m * m);
        srand(1);
        for (int i = 0; i < m; ++i)
            for (int j = 0; j <= i; ++j) {
                double v = (double)rand() / RAND_MAX - 0.5 + (i == j ? 0.01 * i : 0.0);
                hA[(size_t)i * m + j] = hA[(size_t)j * m + i] = v;
            }
        double *A, *A0, *W, *work;
        int *info;
        cudaMalloc(&A, sizeof(double) * m * m);
        cudaMalloc(&A0, sizeof(double) * m * m);
        cudaMalloc(&W, sizeof(double) * m);
        cudaMalloc(&info, sizeof(int));
        cudaMemcpy(A0, hA.data(), sizeof(double) * m * m, cudaMemcpyHostToDevice);
        int lw1 = 0, lw2 = 0, lw3 = 0;
        cusolverDnDsyevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, m, A, m, W, &lw1);
        int meig = 0;
        cusolverDnDsyevdx_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, m, A, m,
                                     0.0, 0.0, m / 2 + 1, m, &meig, W, &lw2);
        syevjInfo_t jp;
        cusolverDnCreateSyevjInfo(&jp);
        cusolverDnXsyevjSetTolerance(jp, 1e-14);
        cusolverDnDsyevj_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, m, A, m, W, &lw3, jp);
        int lw = lw1 > lw2 ? lw1 : lw2;
        lw = lw > lw3 ? lw : lw3;
        cudaMalloc(&work, sizeof(double) * lw);
        auto timeit = [&](const char *name, auto fn) {
            for (int r = 0; r < 2; ++r) {
                cudaMemcpyAsync(A, A0, sizeof(double) * m * m, cudaMemcpyDeviceToDevice, s);
                fn();
            }
            cudaStreamSynchronize(s);
            float best = 1e30f;
            for (int r = 0; r < 5; ++r) {
                cudaMemcpyAsync(A, A0, sizeof(double) * m * m, cudaMemcpyDeviceToDevice, s);
                cudaEventRecord(e0, s);
                fn();
                cudaEventRecord(e1, s);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (ms < best) best = ms;
            }
            int hi;
            cudaMemcpy(&hi, info, sizeof(int), cudaMemcpyDeviceToHost);
            printf("m=%5d %-28s %8.3f ms (info %d)\n", m, name, best, hi);
        };
        timeit("syevd (all)", [&] {
            cusolverDnDsyevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, m, A, m, W, work, lw, info);
        });
        timeit("syevdx (top half)", [&] {
            cusolverDnDsyevdx(h, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, m, A, m, 0.0,
                              0.0, m / 2 + 1, m, &meig, W, work, lw, info);
        });
        timeit("syevj tol 1e-14", [&] {
            cusolverDnDsyevj(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, m, A, m, W, work, lw, info, jp);
        });
        timeit("syevd (values only)", [&] {
            cusolverDnDsyevd(h, CUSOLVER_EIG_MODE_NOVECTOR, CUBLAS_FILL_MODE_LOWER, m, A, m, W, work, lw, info);
        });
        {
            cusolverDnParams_t prm;
            cusolverDnCreateParams(&prm);
            size_t dws = 0, hws = 0;
            cusolverStatus_t bs = cusolverDnXsyevBatched_bufferSize(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, m,
                                                CUDA_R_64F, A, m, CUDA_R_64F, W, CUDA_R_64F, &dws, &hws, 1);
            if (bs == CUSOLVER_STATUS_SUCCESS) {
                void *dw = nullptr;
                cudaMalloc(&dw, dws > 0 ? dws : 16);
                std::vector<char> hw(hws > 0 ? hws : 16);
                timeit("XsyevBatched (batch 1)", [&] {
                    cusolverDnXsyevBatched(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, m, CUDA_R_64F, A, m,
                                           CUDA_R_64F, W, CUDA_R_64F, dw, dws, hw.data(), hws, info, 1);
                });
                cudaFree(dw);
            } else {
                printf("m=%5d XsyevBatched bufferSize status %d\n", m, (int)bs);
            }
            size_t dws2 = 0, hws2 = 0;
            cusolverDnXsyevd_bufferSize(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, m, CUDA_R_64F, A, m,
                                        CUDA_R_64F, W, CUDA_R_64F, &dws2, &hws2);
            void *dw2 = nullptr;
            cudaMalloc(&dw2, dws2 > 0 ? dws2 : 16);
            std::vector<char> hw2(hws2 > 0 ? hws2 : 16);
            timeit("Xsyevd (64-bit API)", [&] {
                cusolverDnXsyevd(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, m, CUDA_R_64F, A, m, CUDA_R_64F,
                                 W, CUDA_R_64F, dw2, dws2, hw2.data(), hws2, info);
            });
            cudaFree(dw2);
            cusolverDnDestroyParams(prm);
        }
        cusolverDnDestroySyevjInfo(jp);
        cudaFree(A); cudaFree(A0); cudaFree(W); cudaFree(work); cudaFree(info);
    }
    return 0;
}
