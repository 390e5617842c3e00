// Does DMMA.8x8x4 give the PTX result when its destination registers alias a source operand?
// PTX semantics: all inputs are read before the outputs are written.  Case B: B operand = d1's input register;
// case A: A operand = d0's input register.  Compared against the same product with distinct registers.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(double* out) {
  const int lane = threadIdx.x;
  double a = 1.0 + lane * 0.25, c0 = 0.5 * lane, c1 = 3.0 - 0.125 * lane;
  // reference: distinct registers
  double r0 = c0, r1 = c1, bsep = c1;
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(r0), "+d"(r1) : "d"(a), "d"(bsep));
  // aliased B: B operand is the d1 register itself
  double x0 = c0, x1 = c1;
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%1}, {%0,%1};" : "+d"(x0), "+d"(x1) : "d"(a));
  // aliased A: A operand is the d0 register itself (C = d0,d1 inputs)
  double y0 = c0, y1 = c1, aref = c0;
  double s0 = c0, s1 = c1;
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(s0), "+d"(s1) : "d"(aref), "d"(a));
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%0}, {%2}, {%0,%1};" : "+d"(y0), "+d"(y1) : "d"(a));
  out[lane * 8 + 0] = r0; out[lane * 8 + 1] = r1; out[lane * 8 + 2] = x0; out[lane * 8 + 3] = x1;
  out[lane * 8 + 4] = s0; out[lane * 8 + 5] = s1; out[lane * 8 + 6] = y0; out[lane * 8 + 7] = y1;
}
int main() {
  double* d; cudaMalloc(&d, 32 * 8 * sizeof(double));
  for (int rep = 0; rep < 3; ++rep) {
    probe<<<1, 32>>>(d);
    double h[256]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    int badB = 0, badA = 0;
    for (int l = 0; l < 32; ++l) {
      badB += h[l * 8 + 2] != h[l * 8 + 0] || h[l * 8 + 3] != h[l * 8 + 1];
      badA += h[l * 8 + 6] != h[l * 8 + 4] || h[l * 8 + 7] != h[l * 8 + 5];
    }
    printf("rep %d: lanes wrong with B aliased to d1: %d, with A aliased to d0: %d (%s)\n", rep, badB, badA,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
