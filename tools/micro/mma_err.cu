// Measures bf16 mma.sync (m16n8k16, fp32 accumulate) dot-product error vs exact (fp64):
// max |tc - exact| / sum|a_i b_i| over random heavy-tailed bf16 vectors, K=256.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_bf16.h>
#include <vector>
__global__ void k(const __nv_bfloat16* A, const __nv_bfloat16* B, float* C, int K) {
  // one warp: C[16x8] = A[16xK] * B[Kx8]; A row-major, B col-major (stored [n][k])
  int l = threadIdx.x;
  float c[4] = {0,0,0,0};
  for (int ks = 0; ks < K; ks += 16) {
    unsigned a[4], b[2];
    int r = l / 4, kk = (l % 4) * 2;
    auto pk = [](__nv_bfloat16 x, __nv_bfloat16 y) { return (unsigned)__bfloat16_as_ushort(x) | ((unsigned)__bfloat16_as_ushort(y) << 16); };
    a[0] = pk(A[r*K+ks+kk], A[r*K+ks+kk+1]);
    a[1] = pk(A[(r+8)*K+ks+kk], A[(r+8)*K+ks+kk+1]);
    a[2] = pk(A[r*K+ks+kk+8], A[r*K+ks+kk+9]);
    a[3] = pk(A[(r+8)*K+ks+kk+8], A[(r+8)*K+ks+kk+9]);
    int n = l / 4;
    b[0] = pk(B[n*K+ks+kk], B[n*K+ks+kk+1]);
    b[1] = pk(B[n*K+ks+kk+8], B[n*K+ks+kk+9]);
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  int r = l / 4, col = (l % 4) * 2;
  C[r*8+col] = c[0]; C[r*8+col+1] = c[1]; C[(r+8)*8+col] = c[2]; C[(r+8)*8+col+1] = c[3];
}
int main() {
  const int K = 256; int trials = 2000;
  __nv_bfloat16 *A, *B; float* C;
  cudaMallocManaged(&A, 16*K*2); cudaMallocManaged(&B, 8*K*2); cudaMallocManaged(&C, 128*4);
  srand(1); double worst = 0, worst_rel_s = 0; double sum_ratio = 0; long cnt = 0;
  for (int t = 0; t < trials; ++t) {
    for (int i = 0; i < 16*K; ++i) { double g = ((rand()/(double)RAND_MAX)*2-1); double m = exp(4.0*((rand()/(double)RAND_MAX)*2-1)); A[i] = __float2bfloat16((float)(g*m)); }
    for (int i = 0; i < 8*K; ++i) { double g = ((rand()/(double)RAND_MAX)*2-1); B[i] = __float2bfloat16((float)g); }
    k<<<1,32>>>(A, B, C, K); cudaDeviceSynchronize();
    for (int r = 0; r < 16; ++r) for (int n = 0; n < 8; ++n) {
      double ex = 0, s = 0;
      for (int i = 0; i < K; ++i) { double p = (double)__bfloat162float(A[r*K+i]) * (double)__bfloat162float(B[n*K+i]); ex += p; s += fabs(p); }
      double e = fabs((double)C[r*8+n] - ex) / s;
      worst = e > worst ? e : worst; sum_ratio += e; ++cnt;
    }
  }
  printf("K=%d max |tc-exact|/sum|ab| = %.3e (= %.2f x 2^-24), mean %.3e\n", K, worst, worst/5.96e-8, sum_ratio/cnt);
  return 0;
}
