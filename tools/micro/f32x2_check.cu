// Compare packed f32x2 add/mul/fma against scalar __fadd_rn/__fmul_rn/__fmaf_rn on random inputs.
#include <cstdio>
#include <cstdint>
#include <cstring>
__device__ __forceinline__ void add2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  asm("{ .reg .b64 a, b, d; mov.b64 a, {%2, %3}; mov.b64 b, {%4, %5}; add.rn.f32x2 d, a, b; mov.b64 {%0, %1}, d; }"
      : "=f"(d0), "=f"(d1) : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
__device__ __forceinline__ void mul2s(float& d0, float& d1, float s, float a0, float a1) {
  asm("{ .reg .b64 a, b, d; mov.b64 a, {%2, %2}; mov.b64 b, {%3, %4}; mul.rn.f32x2 d, a, b; mov.b64 {%0, %1}, d; }"
      : "=f"(d0), "=f"(d1) : "f"(s), "f"(a0), "f"(a1));
}
__device__ __forceinline__ void fma2s0(float& d0, float& d1, float s, float a0, float a1) {
  asm("{ .reg .b64 a, b, c, d; mov.b64 a, {%2, %2}; mov.b64 b, {%3, %4}; mov.b64 c, 0; fma.rn.f32x2 d, a, b, c; mov.b64 {%0, %1}, d; }"
      : "=f"(d0), "=f"(d1) : "f"(s), "f"(a0), "f"(a1));
}
__device__ uint32_t hash(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }
__device__ float rnd(uint32_t i) {
  uint32_t h = hash(i);
  int e = (h >> 23) % 60;  // exponents spanning 2^-30 .. 2^30
  float m = 1.0f + (hash(h) & 0x7fffff) / 8388608.0f;
  float v = ldexpf(m, e - 30);
  return (h & 1) ? -v : v;
}
__global__ void k(unsigned long long* bad, float* ex, float alpha) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  float a0 = rnd(4 * i), a1 = rnd(4 * i + 1), b0 = rnd(4 * i + 2), b1 = rnd(4 * i + 3);
  if (i % 7 == 0) b0 = -a0 * (1.0f + ldexpf(1.0f, -20));  // near-cancellation
  float p0, p1, q0, q1, r0, r1;
  add2(p0, p1, a0, a1, b0, b1);
  mul2s(q0, q1, alpha, a0, a1);
  fma2s0(r0, r1, alpha, a0, a1);
  float sp0 = __fadd_rn(a0, b0), sp1 = __fadd_rn(a1, b1);
  float sq0 = __fmul_rn(alpha, a0), sq1 = __fmul_rn(alpha, a1);
  float sr0 = __fmaf_rn(alpha, a0, 0.f), sr1 = __fmaf_rn(alpha, a1, 0.f);
  int which = -1;
  if (__float_as_uint(p0) != __float_as_uint(sp0) || __float_as_uint(p1) != __float_as_uint(sp1)) which = 0;
  else if (__float_as_uint(q0) != __float_as_uint(sq0) || __float_as_uint(q1) != __float_as_uint(sq1)) which = 1;
  else if (__float_as_uint(r0) != __float_as_uint(sr0) || __float_as_uint(r1) != __float_as_uint(sr1)) which = 2;
  if (which >= 0) {
    unsigned long long c = atomicAdd(&bad[which], 1ull);
    if (c == 0) { float* e = ex + 8 * which; e[0]=a0; e[1]=a1; e[2]=b0; e[3]=b1; e[4]=which==0?p0:which==1?q0:r0; e[5]=which==0?p1:which==1?q1:r1; e[6]=which==0?sp0:which==1?sq0:sr0; e[7]=which==0?sp1:which==1?sq1:sr1; }
  }
}
int main() {
  unsigned long long* bad; float* ex;
  cudaMallocManaged(&bad, 3 * 8); cudaMallocManaged(&ex, 24 * 4);
  memset(bad, 0, 24);
  k<<<1 << 16, 256>>>(bad, ex, 0.9375f);
  cudaDeviceSynchronize();
  const char* nm[3] = {"add.rn.f32x2", "mul.rn.f32x2", "fma.rn.f32x2(+0)"};
  for (int w = 0; w < 3; ++w) {
    printf("%-18s mismatches: %llu of %d\n", nm[w], bad[w], (1 << 24));
    if (bad[w]) printf("   a=(%g,%g) b=(%g,%g) packed=(%.9g,%.9g) scalar=(%.9g,%.9g)\n", ex[8*w], ex[8*w+1], ex[8*w+2], ex[8*w+3], ex[8*w+4], ex[8*w+5], ex[8*w+6], ex[8*w+7]);
  }
  return 0;
}
