// Standalone benchmark + check of the library's FP64 GEMM paths on the
// Kronecker mode-product shapes.
// build (tools/build_gemm_bench.sh):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -o tools/gemm_bench tools/gemm_bench.cu \
//        paper_2406_05020_b200/csrc/{gemm,gemm_tma,pool}.cu
// run: tools/gemm_bench            (TMA kernel, as dispatched by run_gemm)
//      GPFVM_NO_TMA=1 tools/gemm_bench   (cp.async DMMA kernel)
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2406_05020_b200/csrc/internal.h"

namespace gpfvm {
std::atomic<int64_t> g_launches{0};
void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", what, cudaGetErrorString(e)); exit(1); }
}
void set_error(const std::string&) {}
}  // namespace gpfvm
using namespace gpfvm;

__global__ void ref_kernel(Gemm g, int b, double* out) {  // naive reference for batch entry b
  int m = blockIdx.y * blockDim.y + threadIdx.y, n = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= g.M || n >= g.N) return;
  const double* A = g.A + b * g.a_b1;
  const double* B = g.B + b * g.b_b1;
  const double* C = g.C + b * g.c_b1;
  double s = 0;
  for (int sg = 0; sg < g.nseg; sg++)
    for (int k = 0; k < g.K; k++)
      s += A[sg * g.a_sg + m * g.a_rs + k * g.a_cs] * B[sg * g.b_sg + k * g.b_rs + n * g.b_cs];
  out[(int64_t)m * g.N + n] = g.alpha * s + g.beta * C[m * g.c_rs + n * g.c_cs];
}

static void fill_rand(double* d, int64_t n, unsigned seed) {
  std::vector<double> h(n);
  srand(seed);
  for (auto& v : h) v = (double)rand() / RAND_MAX - 0.5;
  cudaMemcpy(d, h.data(), n * 8, cudaMemcpyHostToDevice);
}

// A: M x K (rows a_rs), shared over the batch if a_shared; B row-major (K x N) or column-major; C batch-strided
static void bench(const char* name, int M, int N, int K, int batch, bool brow, bool a_shared, bool b_shared,
                  int nseg = 1, double beta = 0.0, int reps = 10) {
  Gemm g;
  g.M = M; g.N = N; g.K = K; g.nseg = nseg; g.batch1 = batch;
  const int64_t asz1 = (int64_t)M * K * nseg, bsz1 = (int64_t)K * N * nseg, csz1 = (int64_t)M * N;
  const int64_t asz = a_shared ? asz1 : asz1 * batch, bsz = b_shared ? bsz1 : bsz1 * batch, csz = csz1 * batch;
  double *A, *B, *C, *R;
  cudaMalloc(&A, asz * 8); cudaMalloc(&B, bsz * 8); cudaMalloc(&C, csz * 8); cudaMalloc(&R, csz1 * 8);
  fill_rand(A, asz, 1); fill_rand(B, bsz, 2); fill_rand(C, csz, 3);
  g.A = A; g.a_rs = K; g.a_cs = 1; g.a_sg = (int64_t)M * K; g.a_b1 = a_shared ? 0 : asz1;
  if (brow) { g.B = B; g.b_rs = N; g.b_cs = 1; }
  else { g.B = B; g.b_rs = 1; g.b_cs = K; }
  g.b_sg = (int64_t)K * N; g.b_b1 = b_shared ? 0 : bsz1;
  g.C = C; g.c_rs = N; g.c_cs = 1; g.c_b1 = csz1;
  g.beta = beta;
  const int bchk = batch - 1;
  ref_kernel<<<dim3((N + 15) / 16, (M + 15) / 16), dim3(16, 16)>>>(g, bchk, R);
  run_gemm(g, 0);
  cudaDeviceSynchronize();
  std::vector<double> hc(csz1), hr(csz1);
  cudaMemcpy(hc.data(), C + bchk * csz1, csz1 * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(hr.data(), R, csz1 * 8, cudaMemcpyDeviceToHost);
  double err = 0, mx = 0;
  for (int64_t i = 0; i < csz1; i++) { err = fmax(err, fabs(hc[i] - hr[i])); mx = fmax(mx, fabs(hr[i])); }
  g.beta = 0.0;
  for (int i = 0; i < 2; i++) run_gemm(g, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < reps; i++) run_gemm(g, 0);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
  cudaError_t e = cudaGetLastError();
  printf("%-30s M=%5d N=%5d K=%5d seg=%d b=%4d %s: %8.1f us %6.2f TF relerr %.1e %s\n", name, M, N, K, nseg, batch,
         brow ? "Brow" : "Bcol", ms * 1e3, 2.0 * M * N * K * nseg * (double)batch / ms / 1e9, err / mx,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(A); cudaFree(B); cudaFree(C); cudaFree(R);
}

int main(int argc, char** argv) {
  const bool quick = argc > 1;
  // config 1 matvec, forward plan: stage 0 (stacked factor x data, B row-major),
  // stage 1 (data x stacked factor^T, B column-major)
  bench("c1 stage0 T(x)X R=128", 512, 512, 256, 128, true, true, false);
  bench("c1 stage1 Z F^T R=128", 256, 512, 1024, 128, false, false, true);
  if (quick) return 0;
  bench("square Brow", 4096, 4096, 4096, 1, true, true, true, 1, 0.0, 3);
  bench("square Bcol", 4096, 4096, 4096, 1, false, true, true, 1, 0.0, 3);
  bench("c1 stage0 R=1", 512, 512, 256, 1, true, true, false);
  bench("c1 stage1 R=1", 256, 512, 1024, 1, false, false, true);
  bench("beta=1 Bcol", 256, 512, 1024, 16, false, false, true, 1, 1.0);
  bench("beta=1 Brow", 512, 512, 256, 16, true, true, false, 1, 1.0);
  bench("ragged Brow", 1000, 336, 77, 3, true, false, false);
  bench("ragged Bcol", 98, 1002, 514, 2, false, false, false);
  bench("ragged Brow N%16", 200, 338, 100, 5, true, true, false);
  bench("kseg Brow", 256, 256, 64, 8, true, false, true, 3, 0.5);
  bench("kseg Bcol", 192, 256, 40, 8, false, false, true, 3, 0.5);
  bench("c3 stage2 (3D last)", 128 * 256, 256, 256, 1, false, false, true, 2);
  return 0;
}
