// Does mma.sync m16n8k16 (f16 in, f32 acc) multiply fp16 SUBNORMAL A inputs
// exactly on sm_100a?  A = codes masked into exponent-0 halves (c * 2^(sh-24)),
// B = random normal fp16; compare against a double-precision host reference.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_fp16.h>
__device__ void mma(float (&c)[4], const unsigned (&a)[4], unsigned b0, unsigned b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// A row-major 16x16 (halves bits), B col-major 16x8 (B[k][n] at n*16+k), D 16x8
__global__ void k(const unsigned short* A, const unsigned short* B, float* Dout) {
  int lane = threadIdx.x, gid = lane >> 2, t4 = lane & 3;
  unsigned a[4];
  auto ld = [&](int r, int c) { return (unsigned)A[r * 16 + c] | ((unsigned)A[r * 16 + c + 1] << 16); };
  a[0] = ld(gid, 2 * t4); a[1] = ld(gid + 8, 2 * t4); a[2] = ld(gid, 2 * t4 + 8); a[3] = ld(gid + 8, 2 * t4 + 8);
  auto lb = [&](int kk, int n) { return (unsigned)B[n * 16 + kk] | ((unsigned)B[n * 16 + kk + 1] << 16); };
  unsigned b0 = lb(2 * t4, gid), b1 = lb(2 * t4 + 8, gid);
  float c[4] = {0, 0, 0, 0};
  mma(c, a, b0, b1);
  Dout[gid * 8 + 2 * t4] = c[0]; Dout[gid * 8 + 2 * t4 + 1] = c[1];
  Dout[(gid + 8) * 8 + 2 * t4] = c[2]; Dout[(gid + 8) * 8 + 2 * t4 + 1] = c[3];
}
static float h2f(unsigned short h) { __half x; memcpy(&x, &h, 2); return __half2float(x); }
int main() {
  unsigned short *A, *B; float* D;
  cudaMallocManaged(&A, 512); cudaMallocManaged(&B, 256); cudaMallocManaged(&D, 512);
  srand(1);
  for (int mode = 0; mode < 2; ++mode) {
  double worst = 0; long bad = 0, tot = 0;
  for (int trial = 0; trial < 2000; ++trial) {
    int sh = trial % 7;  // field shift 0..6
    int bits = (trial / 7) % 2 ? 4 : 2;
    for (int i = 0; i < 256; ++i) {
      unsigned code = rand() & ((1u << bits) - 1);
      if (mode == 0) {
        A[i] = (unsigned short)(code << sh);  // exponent 0: subnormal c*2^(sh-24)
      } else {
        __half hc = __float2half((float)code); memcpy(&A[i], &hc, 2);  // normal exact code
      }
    }
    for (int i = 0; i < 128; ++i) {
      float v = ((rand() / (float)RAND_MAX) - 0.5f) * 8.f;
      __half h = __float2half_rn(v); memcpy(&B[i], &h, 2);
    }
    k<<<1, 32>>>(A, B, D); cudaDeviceSynchronize();
    for (int m = 0; m < 16; ++m) for (int n = 0; n < 8; ++n) {
      double ref = 0;
      for (int kk = 0; kk < 16; ++kk) ref += (double)h2f(A[m * 16 + kk]) * (double)h2f(B[n * 16 + kk]);
      double got = D[m * 8 + n];
      double scale = 0; for (int kk = 0; kk < 16; ++kk) scale += fabs((double)h2f(A[m*16+kk]) * h2f(B[n*16+kk]));
      double rel = scale > 0 ? fabs(got - ref) / scale : fabs(got - ref);
      if (rel > worst) worst = rel;
      if (rel > 1e-6) ++bad;
      ++tot;
    }
  }
  printf("%s-A mma: worst rel err %.3e, %ld of %ld outputs off by > 1e-6\n", mode ? "normal" : "subnormal", worst, bad, tot);
  }
  // sanity: a single product, smallest subnormal times 1.0
  for (int i = 0; i < 256; ++i) A[i] = 0; for (int i = 0; i < 128; ++i) B[i] = 0;
  A[0] = 1; __half one = __float2half(1.0f); memcpy(&B[0], &one, 2);
  k<<<1, 32>>>(A, B, D); cudaDeviceSynchronize();
  printf("2^-24 * 1 = %.6e (expect %.6e)\n", D[0], ldexp(1.0, -24));
  return 0;
}
