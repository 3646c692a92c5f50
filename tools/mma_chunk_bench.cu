// Standalone efficiency of k_condense's mma_chunk (one 64x64 output tile per 4-warp CTA, [64][16]
// k-chunks in shared memory, TMA 128-byte swizzle layout) with and without a CTA barrier per chunk.
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/mma_chunk_bench.cu -o /tmp/mb -lcuda
#include <cstdio>
#include "../paper_2312_12771_b200/csrc/condense.cu"
template <int SYNC>
__global__ void __launch_bounds__(128) kb(double* out, int iters) {
  __shared__ __align__(1024) double st[2][2 * 64 * hom::KC];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < 2 * 2 * 64 * hom::KC; i += 128) (&st[0][0])[i] = 1e-3 * (i % 97);
  __syncthreads();
  double acc[4][4][2] = {};
  const int R0 = (warp >> 1) * 32, C0 = (warp & 1) * 32;
  for (int it = 0; it < iters; ++it) {
    const double* s = st[it & 1];
    hom::mma_chunk<false, true>(acc, s, s + 64 * hom::KC, R0, C0, lane);
    if (SYNC) __syncthreads();
  }
  double v = 0;
  for (int a = 0; a < 4; ++a) for (int b = 0; b < 4; ++b) v += acc[a][b][0] + acc[a][b][1];
  if (v == 1.2345) out[0] = v;
}
template <int SYNC>
void run(int ctas_per_sm, int iters) {
  double* o; cudaMalloc(&o, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int grid = 148 * ctas_per_sm;
  kb<SYNC><<<grid, 128>>>(o, 10);
  cudaEventRecord(e0);
  kb<SYNC><<<grid, 128>>>(o, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = (double)grid * iters * 2.0 * 64 * 64 * hom::KC;
  printf("sync %d ctas/SM %d: %.2f TFLOP/s (%s)\n", SYNC, ctas_per_sm, fl / (ms * 1e-3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
}
int main() {
  for (int c : {1, 2, 3, 4}) { run<0>(c, 20000); run<1>(c, 20000); }
  return 0;
}
