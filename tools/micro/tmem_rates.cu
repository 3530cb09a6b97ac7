// TMEM as plain per-warp storage (no MMA): tcgen05.ld/st throughput and latency with
// 8 warps per SM, the lane-quarter rule for an 8-warp CTA, runtime column offsets.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_rates tools/micro/tmem_rates.cu && ./tmem_rates
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ void st32(uint32_t taddr, const float (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
        "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
        "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]), "f"(v[17]), "f"(v[18]),
        "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]),
        "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
        : "memory");
}
__device__ __forceinline__ void ld32(uint32_t taddr, float (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]), "=f"(v[8]),
          "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15]), "=f"(v[16]),
          "=f"(v[17]), "=f"(v[18]), "=f"(v[19]), "=f"(v[20]), "=f"(v[21]), "=f"(v[22]), "=f"(v[23]), "=f"(v[24]),
          "=f"(v[25]), "=f"(v[26]), "=f"(v[27]), "=f"(v[28]), "=f"(v[29]), "=f"(v[30]), "=f"(v[31])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void ld4(uint32_t taddr, float (&v)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]) : "r"(taddr) : "memory");
}
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// mode 0: st+ld throughput (x32 each per round), mode 1: ld only, mode 2: st only, 3: latency chain
__global__ void __launch_bounds__(256, 1) k(int mode, int rounds, float* out, long long* cyc, int* chk) {
    __shared__ uint32_t base;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    // warp w: lanes 32*(w%4), columns 256*(w/4)
    const uint32_t t = base + ((uint32_t)(32 * (warp & 3)) << 16) + 256u * (warp >> 2);
    float v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = (float)(threadIdx.x * 100 + j + blockIdx.x);
    // correctness: write 8 slots, read back with runtime offsets
    for (int s = 0; s < 8; ++s) {
        float w[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) w[j] = v[j] + 1000.f * s;
        st32(t + 32 * s, w);
    }
    wait_st();
    int bad = 0;
    for (int s = 0; s < 8; ++s) {
        const int off = (s * 3 + (int)blockIdx.x * 5) & 28;  // runtime (warp-uniform), multiple of 4
        float w[4];
        ld4(t + 32 * s + off, w);
        wait_ld();
        for (int i = 0; i < 4; ++i) bad += w[i] != v[off + i] + 1000.f * s;
    }
    if (bad) atomicAdd(chk, bad);
    __syncwarp();
    long long c0 = clock64();
    float acc = 0.f;
    if (mode == 3) {
        float x = v[0];
        for (int r = 0; r < rounds; ++r) {
            float w[4];
            ld4(t + ((__float_as_uint(x) & 0) ), w);
            wait_ld();
            x = w[0];
            v[0] = x + 1.f;
            // dependent store of one column to keep the chain honest
            asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(t), "f"(v[0]) : "memory");
            wait_st();
        }
        acc = x;
    } else {
        for (int r = 0; r < rounds; ++r) {
            const uint32_t a = t + 32 * (r & 7);
            if (mode != 1) st32(a, v);
            if (mode != 2) {
                ld32(a ^ 32, v);
                wait_ld();
            }
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] += 1.f;
        }
        wait_st();
#pragma unroll
        for (int j = 0; j < 32; ++j) acc += v[j];
    }
    long long c1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (lane == 0) cyc[blockIdx.x * 8 + warp] = c1 - c0;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    long long* cyc;
    int* chk;
    cudaMalloc(&out, nsm * 256 * 4);
    cudaMalloc(&cyc, nsm * 8 * 8);
    cudaMalloc(&chk, 4);
    cudaMemset(chk, 0, 4);
    const char* names[] = {"st.x32+ld.x32", "ld.x32", "st.x32", "ld.x4+st.x1 latency chain"};
    for (int mode = 0; mode < 4; ++mode) {
        const int rounds = mode == 3 ? 2000 : 4000;
        k<<<nsm, 256>>>(mode, rounds, out, cyc, chk);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("mode %d: %s\n", mode, cudaGetErrorString(e));
            return 1;
        }
        long long h[8];
        cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < 8; ++i) avg += h[i] / 8.0;
        const double per = avg / rounds;
        int c = 0;
        cudaMemcpy(&c, chk, 4, cudaMemcpyDeviceToHost);
        if (mode == 3)
            printf("%-28s %.1f cycles per round (1 warp view, 8 warps/SM)  readback errors %d\n", names[mode], per, c);
        else {
            const double bytes = (mode == 0 ? 2 : 1) * 32.0 * 32 * 4 * 8;  // per round, whole SM (8 warps)
            printf("%-28s %.1f cycles per round per warp; SM-wide %.0f B/clk  readback errors %d\n", names[mode], per,
                   bytes / per, c);
        }
    }
    return 0;
}
