// Does a kernel that uses tcgen05.alloc get more than one resident CTA per SM?
// nvcc -gencode arch=compute_100a,code=sm_100a -o tmem_occ tools/micro/tmem_occupancy.cu && ./tmem_occ
#include <cstdio>
#include <cstdint>
template <bool TM>
__global__ void __launch_bounds__(256, 2) k(int* out) {
    extern __shared__ uint32_t s[];
    if constexpr (TM) {
        if ((threadIdx.x >> 5) == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
                (uint32_t)__cvta_generic_to_shared(s)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
        __syncthreads();
        if ((threadIdx.x >> 5) == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(s[0]));
    }
    if (threadIdx.x == 0) out[blockIdx.x] = s[1];
}
int main() {
    for (int smem : {60000, 100000, 108576}) {
        int a = 0, b = 0;
        cudaFuncSetAttribute(k<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(k<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k<false>, 256, smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k<true>, 256, smem);
        printf("smem %d: without tcgen05.alloc %d CTAs/SM, with %d\n", smem, a, b);
    }
    return 0;
}
