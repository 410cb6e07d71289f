// Where does a kernel's dynamic shared memory start (shared-window address)?
// The tcgen05 kernels align their tiles to 1024 B; this prints the raw base.
#include <cstdio>
#include <cstdint>
__global__ void k(uint32_t *out) {
    extern __shared__ uint8_t s[];
    if (threadIdx.x == 0) out[blockIdx.x] = (uint32_t)__cvta_generic_to_shared(s);
}
int main() {
    uint32_t *d, h[4];
    cudaMalloc(&d, 16);
    for (int bytes : {1024, 100000, 232448 - 1024, 232448}) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        k<<<4, 640, bytes>>>(d);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("dyn %6d B: %s base 0x%x 0x%x (mod 1024 = %u)\n", bytes, cudaGetErrorString(e), h[0], h[1], h[0] % 1024);
    }
    int v;
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
    printf("max dyn smem per block optin %d\n", v);
    return 0;
}
