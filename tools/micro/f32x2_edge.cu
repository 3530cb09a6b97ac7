// Edge classes for packed f32x2 vs scalar: exact cancellation, zeros of both signs, subnormals, huge.
#include <cstdio>
#include <cstdint>
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
__global__ void k(const float* a, const float* b, int n, float alpha, unsigned* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x; if (i >= n) return;
  float p0,p1,q0,q1,r0,r1;
  add2(p0,p1,a[i],a[i],b[i],b[i]); mul2s(q0,q1,alpha,a[i],b[i]); fma2s0(r0,r1,alpha,a[i],b[i]);
  out[6*i+0]=__float_as_uint(p0)^__float_as_uint(__fadd_rn(a[i],b[i]));
  out[6*i+1]=__float_as_uint(q0)^__float_as_uint(__fmul_rn(alpha,a[i]));
  out[6*i+2]=__float_as_uint(q1)^__float_as_uint(__fmul_rn(alpha,b[i]));
  out[6*i+3]=__float_as_uint(r0)^__float_as_uint(__fmaf_rn(alpha,a[i],0.f));
  out[6*i+4]=__float_as_uint(r1)^__float_as_uint(__fmaf_rn(alpha,b[i],0.f));
  out[6*i+5]=__float_as_uint(p0);
}
int main() {
  const float vals[] = {0.f, -0.f, 1.f, -1.f, 3.5f, -3.5f, 1e-38f, -1e-38f, 1e-40f, -1e-40f, 1e-45f, 1e30f, -1e30f, 3e38f, -3e38f, 0.5f};
  const int nv = sizeof(vals)/4; int n = nv*nv;
  float *a, *b; unsigned* o; cudaMallocManaged(&a,n*4); cudaMallocManaged(&b,n*4); cudaMallocManaged(&o,n*24);
  for (int i=0;i<nv;++i) for (int j=0;j<nv;++j) { a[i*nv+j]=vals[i]; b[i*nv+j]=vals[j]; }
  k<<<(n+127)/128,128>>>(a,b,n,0.9375f,o); cudaDeviceSynchronize();
  const char* nm[5]={"add2","mul2.a","mul2.b","fma2.a","fma2.b"}; int bad=0;
  for (int i=0;i<n;++i) for (int w=0;w<5;++w) if (o[6*i+w]) { if (bad<30) printf("%s a=%g b=%g packed^scalar=%08x (packed add=%08x)\n", nm[w], a[i], b[i], o[6*i+w], o[6*i+5]); ++bad; }
  printf("edge mismatches: %d\n", bad);
}
