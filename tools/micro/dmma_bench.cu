// Microbenchmark: FP64 tensor (mma.sync m8n8k4 f64) vs FP64 FMA throughput on this GPU.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dmma(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0001;
    double c[8][2];
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
        }
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.0) out[0] = s;
}

__global__ void k_dfma(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0001;
    double c[16];
    for (int i = 0; i < 16; ++i) c[i] = i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) c[i] = fma(c[i], b, a);
    }
    double s = 0;
    for (int i = 0; i < 16; ++i) s += c[i];
    if (s == 12345.0) out[0] = s;
}

int main() {
    double* d;
    cudaMalloc(&d, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096;
    for (int warps : {4, 8, 16}) {
        dim3 grid(sms * 4), block(32 * warps);
        k_dmma<<<grid, block>>>(d, 16);
        cudaEventRecord(e0);
        k_dmma<<<grid, block>>>(d, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double macs = (double)grid.x * warps * iters * 8 * 256;
        printf("DMMA warps/blk=%d: %.2f TFLOP/s (fp64 MMA)\n", warps, 2 * macs / ms / 1e9);
        k_dfma<<<grid, block>>>(d, 16);
        cudaEventRecord(e0);
        k_dfma<<<grid, block>>>(d, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        macs = (double)grid.x * block.x * iters * 16;
        printf("DFMA warps/blk=%d: %.2f TFLOP/s (fp64 FMA)\n", warps, 2 * macs / ms / 1e9);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
