// Standalone benchmark + check of the DMMA GEMM used by libgpfvm
// (build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o gemm_bench tools/gemm_bench.cu)
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2406_05020_b200/csrc/gemm.cu"

namespace gpfvm {
std::atomic<int64_t> g_launches{0};
void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", what, cudaGetErrorString(e)); exit(1); }
}
void set_error(const std::string&) {}
}  // namespace gpfvm
using namespace gpfvm;

__global__ void ref_kernel(Gemm g, double* out) {  // naive reference for batch 0
  int m = blockIdx.y * blockDim.y + threadIdx.y, n = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= g.M || n >= g.N) return;
  double s = 0;
  for (int k = 0; k < g.K; k++) s += g.A[m * g.a_rs + k * g.a_cs] * g.B[k * g.b_rs + n * g.b_cs];
  out[(int64_t)m * g.N + n] = s;
}

static void bench(const char* name, int M, int N, int K, int batch, bool brow, int reps = 10) {
  int64_t asz = (int64_t)M * K * batch, bsz = (int64_t)K * N * batch, csz = (int64_t)M * N * batch;
  double *A, *B, *C, *R;
  cudaMalloc(&A, asz * 8); cudaMalloc(&B, bsz * 8); cudaMalloc(&C, csz * 8); cudaMalloc(&R, (int64_t)M * N * 8);
  std::vector<double> h(std::max(asz, bsz));
  for (auto& v : h) v = (double)rand() / RAND_MAX - 0.5;
  cudaMemcpy(A, h.data(), asz * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(B, h.data(), bsz * 8, cudaMemcpyHostToDevice);
  Gemm g;
  g.M = M; g.N = N; g.K = K; g.batch1 = batch;
  g.A = A; g.a_rs = K; g.a_cs = 1; g.a_b1 = (int64_t)M * K;
  if (brow) { g.B = B; g.b_rs = N; g.b_cs = 1; }
  else { g.B = B; g.b_rs = 1; g.b_cs = K; }
  g.b_b1 = (int64_t)K * N;
  g.C = C; g.c_rs = N; g.c_cs = 1; g.c_b1 = (int64_t)M * N;
  run_gemm(g, 0);
  ref_kernel<<<dim3((N + 15) / 16, (M + 15) / 16), dim3(16, 16)>>>(g, R);
  cudaDeviceSynchronize();
  std::vector<double> hc((int64_t)M * N), hr((int64_t)M * N);
  cudaMemcpy(hc.data(), C, hc.size() * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(hr.data(), R, hr.size() * 8, cudaMemcpyDeviceToHost);
  double err = 0, mx = 0;
  for (size_t i = 0; i < hc.size(); i++) { err = fmax(err, fabs(hc[i] - hr[i])); mx = fmax(mx, fabs(hr[i])); }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < reps; i++) run_gemm(g, 0);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
  printf("%-34s M=%6d N=%6d K=%7d b=%4d %s: %8.1f us  %6.2f TF  relerr %.1e\n", name, M, N, K, batch,
         brow ? "Brow" : "Bcol", ms * 1e3, 2.0 * M * N * K * batch / ms / 1e9, err / mx);
  cudaFree(A); cudaFree(B); cudaFree(C); cudaFree(R);
}

int main() {
  bench("square", 4096, 4096, 4096, 1, true, 3);
  bench("square", 4096, 4096, 4096, 1, false, 3);
  bench("c1 x-stage R=128 (X F^T)", 256, 512, 512, 128, false);
  bench("c1 t-stage R=128 (T Z)", 256, 512, 256, 128, true);
  bench("c1 x-stage R=1", 256, 512, 512, 1, false);
  bench("c1 t-stage R=1", 256, 512, 256, 1, true);
  bench("schur S -= Gpb^T Y", 1024, 1024, 131072, 1, false, 3);
  bench("predict Sinv Z", 1024, 65536, 1024, 1, true, 3);
  bench("ragged", 1000, 333, 77, 3, true);
  bench("ragged col", 97, 1001, 513, 2, false);
  return 0;
}
