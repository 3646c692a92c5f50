// FP64 peak microbenchmarks on sm_100a: DFMA (CUDA-core) vs DMMA (mma.sync .f64) shapes.
// Used once to pick the condensation kernel's math path; results go to profiles/.
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096

__global__ void dfma_kernel(double* out, double a, double b) {
  double acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i];
  if (s == 1234.5) out[0] = s;
}

__global__ void dmma_m8n8k4(double* out, double a0, double b0) {
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  double a = a0 + threadIdx.x * 1e-9, b = b0;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 1234.5) out[0] = s;
}

__global__ void dmma_m16n8k4(double* out, double a0, double b0) {
  double c[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  double a = a0 + threadIdx.x * 1e-9, b = b0;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a), "d"(b), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 1234.5) out[0] = s;
}

__global__ void dmma_m16n8k8(double* out, double a0, double b0) {
  double c[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  double a = a0 + threadIdx.x * 1e-9, b = b0;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a), "d"(b), "d"(a), "d"(b), "d"(b), "d"(a));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 1234.5) out[0] = s;
}

__global__ void dmma_m16n8k16(double* out, double a0, double b0) {
  double c[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  double a = a0 + threadIdx.x * 1e-9, b = b0;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a), "d"(b), "d"(a), "d"(b), "d"(a), "d"(b), "d"(a), "d"(b),
                     "d"(b), "d"(a), "d"(b), "d"(a));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 1234.5) out[0] = s;
}

template <typename K>
static void run(const char* name, K kern, double flop_per_thread_iter, int blocks_per_sm, int threads) {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  double* out; cudaMalloc(&out, 8);
  int grid = p.multiProcessorCount * blocks_per_sm;
  for (int w = 0; w < 3; ++w) kern<<<grid, threads>>>(out, 1.0000001, 1e-7);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    for (int k = 0; k < 5; ++k) kern<<<grid, threads>>>(out, 1.0000001, 1e-7);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  double flops = 5.0 * grid * threads * (double)ITERS * flop_per_thread_iter;
  printf("%-14s grid=%d thr=%d  %.2f TFLOP/s  (%.3f ms / 5 launches) err=%s\n", name, grid, threads,
         flops / (best * 1e-3) / 1e12, best, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("device %s SMs=%d clock=%d kHz\n", p.name, p.multiProcessorCount, p.clockRate);
  for (int bps : {2, 4, 8}) {
    run("dfma", dfma_kernel, 8 * 2.0, bps, 256);
    run("dmma_m8n8k4", dmma_m8n8k4, 8 * 512.0 / 32, bps, 256);
    run("dmma_m16n8k4", dmma_m16n8k4, 4 * 1024.0 / 32, bps, 256);
    run("dmma_m16n8k8", dmma_m16n8k8, 4 * 2048.0 / 32, bps, 256);
    run("dmma_m16n8k16", dmma_m16n8k16, 4 * 4096.0 / 32, bps, 256);
  }
  return 0;
}
