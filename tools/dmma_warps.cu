// DMMA (mma.sync.m8n8k4.f64) throughput vs resident warps per SM sub-partition: one CTA per SM,
// W warps, every warp issues independent accumulator chains (NACC per warp) from registers.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/dmma_warps.cu -o /tmp/dw && /tmp/dw
#include <cstdio>
template <int NACC>
__global__ void k(double* out, int iters) {
  double acc[NACC][2];
  double a = threadIdx.x * 1e-3, b = blockIdx.x * 1e-3;
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i][0] = acc[i][1] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.0) out[0] = s;
}
template <int NACC>
void run(int warps, int iters) {
  double* o;
  cudaMalloc(&o, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<NACC><<<148, 32 * warps>>>(o, 10);
  cudaEventRecord(e0);
  k<NACC><<<148, 32 * warps>>>(o, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = 148.0 * warps * iters * NACC * 512.0;
  printf("warps/SM %2d (per SMSP %.2f) NACC %2d: %.2f TFLOP/s\n", warps, warps / 4.0, NACC, fl / (ms * 1e-3) / 1e12);
  cudaFree(o);
}
int main() {
  for (int w : {4, 8, 12, 16, 32}) { run<16>(w, 20000); }
  for (int w : {4, 8}) { run<4>(w, 40000); run<8>(w, 40000); run<32>(w, 10000); }
  return 0;
}
