// Per-SM throughput of the PE's instructions on this B200: 8 independent chains per thread,
// 4..32 warps per SM, clock64 cycles. Prints warp-instructions per clock per SM.
#include <cstdio>
#define ITERS 4096
template <int OP>
__global__ void bench(float* out, long long* cyc, float a) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("min.xorsign.abs.f32 %0, %0, %1;" : "+f"(x[i]) : "f"(a));
      if (OP == 1) asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(x[i]) : "f"(a));
      if (OP == 2) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(x[i]) : "f"(a));
      if (OP == 3) asm volatile("{ .reg .b64 v, s; mov.b64 v, {%0, %0}; mov.b64 s, {%1, %1}; add.rn.f32x2 v, v, s; mov.b64 {%0, %0}, v; }" : "+f"(x[i]) : "f"(a));
      if (OP == 4) { unsigned u = __float_as_uint(x[i]); asm volatile("shf.l.wrap.b32 %0, %1, %0, 1;" : "+r"(u) : "r"(__float_as_uint(a))); x[i] = __uint_as_float(u); }
      if (OP == 5) asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(x[i]) : "f"(a));
    }
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int OP> void run(const char* nm, int warps) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; long long* cyc; cudaMalloc(&out, sms * warps * 32 * 4); cudaMallocManaged(&cyc, sms * 8);
  bench<OP><<<sms, warps * 32>>>(out, cyc, 0.9375f);
  bench<OP><<<sms, warps * 32>>>(out, cyc, 0.9375f);
  cudaDeviceSynchronize();
  double c = 0; for (int i = 0; i < sms; ++i) c += cyc[i]; c /= sms;
  double instr = (double)warps * ITERS * 8;  // warp-instructions per SM (f32x2 counts once)
  printf("%-26s warps/SM %2d : %.2f warp-inst/clk/SM\n", nm, warps, instr / c);
  cudaFree(out); cudaFree(cyc);
}
int main() {
  for (int w : {4, 8, 16, 32}) {
    run<0>("FMNMX.XORSIGN", w); run<1>("FMUL", w); run<2>("FADD", w); run<3>("FADD2 (f32x2)", w);
    run<4>("SHF.L.W (funnel)", w); run<5>("FFMA", w);
  }
}
