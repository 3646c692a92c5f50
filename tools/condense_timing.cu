// Phase timing of k_condense on synthetic SPD tiles (clock64 marks, HOM_TIMING build).
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -DHOM_TIMING tools/condense_timing.cu -o /tmp/ct
// ./ct NT NB   -> per-column averages over the first 64 CTAs of: diagonal accumulate, diagonal
// factor + inverse, Y_J + Schur accumulation, off-diagonal tiles (accumulate + TRSM).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2312_12771_b200/csrc/condense.cu"

int main(int argc, char** argv) {
  int nt = argc > 1 ? atoi(argv[1]) : 8, nb = argc > 2 ? atoi(argv[2]) : 4096;
  size_t tiles = (size_t)nt * (nt + 1) / 2;
  size_t per = tiles * hom::TILE_ELEMS;
  std::vector<double> h(per);
  // SPD: tridiagonal-ish 2 on the diagonal, -0.5 coupling to neighbours, as dense lower tiles
  int n = nt * 64;
  for (int I = 0; I < nt; ++I)
    for (int J = 0; J <= I; ++J)
      for (int r = 0; r < 64; ++r)
        for (int c = 0; c < 64; ++c) {
          int i = I * 64 + r, j = J * 64 + c;
          double v = (i == j) ? 4.0 : ((i - j == 1 || i - j == 37) ? -0.5 : 0.0);
          if (I == nt - 1 && j < 5 && i != j) v = 0.01;
          h[(size_t)(I * (I + 1) / 2 + J) * 4096 + r * 64 + c] = v;
        }
  double *Kt, *Y, *Cavg, *Ceff, *X;
  int* info;
  cudaMalloc(&Kt, per * nb * 8);
  for (int b = 0; b < nb; ++b) cudaMemcpy(Kt + per * b, h.data(), per * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&Y, (size_t)n * 8 * nb * 8);
  cudaMemset(Y, 0, (size_t)n * 8 * nb * 8);
  cudaMalloc(&Cavg, 64 * nb * 8);
  cudaMemset(Cavg, 0, 64 * nb * 8);
  cudaMalloc(&Ceff, 64 * nb * 8);
  cudaMalloc(&X, (size_t)n * 8 * nb * 8);
  cudaMalloc(&info, nb * 4);
  cudaMemset(info, 0, nb * 4);
  hom::RveDev R{};
  R.dim = 2; R.nt = nt; R.NT = n; R.npad = n; R.m = 3; R.ncol = 3; R.vol = 1.0;
  {  // dense tile structure: every lower tile processed, slot I(I+1)/2 + J
    std::vector<int> ts((size_t)nt * nt, -1);
    std::vector<uint8_t> gz((size_t)nt * nt, 0);
    for (int I = 0; I < nt; ++I)
      for (int J = 0; J <= I; ++J) { ts[(size_t)I * nt + J] = I * (I + 1) / 2 + J; gz[(size_t)I * nt + J] = 1; }
    int* dts; uint8_t* dgz;
    cudaMalloc(&dts, ts.size() * 4); cudaMemcpy(dts, ts.data(), ts.size() * 4, cudaMemcpyHostToDevice);
    cudaMalloc(&dgz, gz.size()); cudaMemcpy(dgz, gz.data(), gz.size(), cudaMemcpyHostToDevice);
    R.tslot = dts; R.g_nz = dgz; R.tile_nz = dgz; R.nslot = (int)tiles; R.xb0 = 0; R.dense_tiles = 1;
  }
  std::vector<double> hk(per * nb);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  hom::launch_condense(R, 0, nb, Kt, Y, Cavg, nullptr, Ceff, nullptr, nullptr, X, info, 0);
  cudaDeviceSynchronize();
  for (int b = 0; b < nb; ++b) cudaMemcpy(Kt + per * b, h.data(), per * 8, cudaMemcpyHostToDevice);
  cudaEventRecord(e0);
  hom::launch_condense(R, 0, nb, Kt, Y, Cavg, nullptr, Ceff, nullptr, nullptr, X, info, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("nt=%d nb=%d  kernel %.3f ms  err=%s\n", nt, nb, ms, cudaGetErrorString(cudaGetLastError()));
  static long long tm[64][40][8];
  cudaMemcpyFromSymbol(tm, hom::g_tm, sizeof(tm));
  const char* var = getenv("HOM_CONDENSE");
  if (var && var[0] == 'w') {  // k_condense_ws marks: MMA 0..4, factor warp 5..7
    printf("  J |  syrk | accum+park | waitG | trsm | total || factor: waitS chain  Y+store (k-cycles)\n");
    double t[8] = {};
    for (int J = 0; J < nt && J < 40; ++J) {
      double v[8] = {};
      for (int b = 0; b < 64; ++b) {
        long long* m = tm[b][J];
        v[0] += m[1] - m[0]; v[1] += m[2] - m[1]; v[2] += m[3] - m[2]; v[3] += m[4] - m[3]; v[4] += m[4] - m[0];
        v[5] += m[5] - (J ? tm[b][J - 1][7] : m[0]); v[6] += m[6] - m[5]; v[7] += m[7] - m[6];
      }
      printf("%3d | %5.1f | %10.1f | %5.1f | %4.1f | %5.1f || %5.1f %6.1f %6.1f\n", J, v[0] / 64e3, v[1] / 64e3,
             v[2] / 64e3, v[3] / 64e3, v[4] / 64e3, v[5] / 64e3, v[6] / 64e3, v[7] / 64e3);
      for (int k = 0; k < 8; ++k) t[k] += v[k];
    }
    printf("sum | %5.1f | %10.1f | %5.1f | %4.1f | %5.1f || %5.1f %6.1f %6.1f\n", t[0] / 64e3, t[1] / 64e3, t[2] / 64e3,
           t[3] / 64e3, t[4] / 64e3, t[5] / 64e3, t[6] / 64e3, t[7] / 64e3);
    return 0;
  }
  printf("  J |  diagS | factor |   Y+Sacc | offdiag | total | (k-cycles, mean over 64 CTAs)\n");
  double tot[5] = {};
  for (int J = 0; J < nt && J < 40; ++J) {
    double v[5] = {};
    for (int b = 0; b < 64; ++b) {
      long long* m = tm[b][J];
      v[0] += m[1] - m[0]; v[1] += m[2] - m[1]; v[2] += m[3] - m[2]; v[3] += m[4] - m[3]; v[4] += m[4] - m[0];
    }
    printf("%3d | %6.1f | %6.1f | %8.1f | %7.1f | %5.1f\n", J, v[0] / 64e3, v[1] / 64e3, v[2] / 64e3, v[3] / 64e3,
           v[4] / 64e3);
    for (int k = 0; k < 5; ++k) tot[k] += v[k];
  }
  printf("sum | %6.1f | %6.1f | %8.1f | %7.1f | %5.1f\n", tot[0] / 64e3, tot[1] / 64e3, tot[2] / 64e3, tot[3] / 64e3,
         tot[4] / 64e3);
  {  // inside the factor: first chol16 (+ its barrier), the blocked loop, the off-diagonal inverse
    double f[3] = {};
    for (int J = 0; J < nt && J < 40; ++J)
      for (int b = 0; b < 64; ++b) {
        long long* m = tm[b][J];
        f[0] += m[5] - m[1]; f[1] += m[6] - m[1]; f[2] += m[2] - m[6];
      }
    printf("factor split (k-cycles summed over J): chol16(0) %.1f | 4-block loop %.1f | inverse %.1f\n",
           f[0] / 64e3, f[1] / 64e3, f[2] / 64e3);
    double bw = 0.0;
    for (int b = 0; b < 64; ++b) bw += tm[b][39][1] - tm[b][39][0];
    printf("backward X = G^-T Y (k-cycles, after the C_eff epilogue): %.1f\n", bw / 64e3);
  }
  return 0;
}
