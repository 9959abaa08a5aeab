// Standalone check of the bulk-copy ring used by k_band_dft's fold.
#include <cstdio>
#include <cstdint>
#include <vector>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile("{\n.reg .pred done;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n@!done bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b)) : "memory");
}
__global__ void k(const double2* x, double2* y, int n) {
    extern __shared__ __align__(128) double2 buf[];
    __shared__ __align__(8) uint64_t bar[1];
    if (threadIdx.x == 0) { mbar_init(&bar[0], 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    __syncthreads();
    if (threadIdx.x == 0) { mbar_expect_tx(&bar[0], n * 16); bulk_g2s(buf, x, n * 16, &bar[0]); }
    mbar_wait(&bar[0], 0);
    for (int i = threadIdx.x; i < n; i += blockDim.x) y[i] = buf[i];
}
int main() {
    const int n = 256;
    std::vector<double2> h(n);
    for (int i = 0; i < n; ++i) h[i] = make_double2(i, -i);
    double2 *dx, *dy;
    cudaMalloc(&dx, n * 16); cudaMalloc(&dy, n * 16);
    cudaMemcpy(dx, h.data(), n * 16, cudaMemcpyHostToDevice);
    cudaMemset(dy, 0, n * 16);
    k<<<1, 128, n * 16>>>(dx, dy, n);
    printf("launch %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    cudaMemcpy(h.data(), dy, n * 16, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < n; ++i) bad += h[i].x != i || h[i].y != -i;
    printf("bad %d  y[5]=%g\n", bad, h[5].x);
}
