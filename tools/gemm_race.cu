// Two-stream reproducer for the concurrency failure of DESIGN.md §4.4: stream A
// repeats one TMA GEMM (bitwise compared with its own first, solitary result),
// stream B keeps the machine busy with GEMMs the TMA path rejects (cp.async
// kernel) or, with mode 1, with other TMA GEMMs, mode 2: nothing (control).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/gemm_race tools/gemm_race.cu \
//        paper_2406_05020_b200/csrc/{gemm,gemm_tma,pool}.cu
// run:   tools/gemm_race [mode] [reps]
#include <cstdio>
#include <cstdlib>
#include <cstring>
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

static double* dalloc(int64_t n, unsigned seed) {
  double* p;
  cudaMalloc(&p, n * 8);
  std::vector<double> h(n);
  srand(seed);
  for (auto& v : h) v = (double)rand() / RAND_MAX - 0.5;
  cudaMemcpy(p, h.data(), n * 8, cudaMemcpyHostToDevice);
  return p;
}

// mode 3: a kernel with the cp.async GEMM's footprint (128 threads, 38 KB of
// dynamic shared memory, 288 CTAs) that never issues cp.async
__global__ void dummy_smem_kernel(const double* __restrict__ in, double* out, int n) {
  extern __shared__ double sm[];
  const int words = 38912 / 8;
  double acc = 0.0;
  for (int it = 0; it < 40; it++) {
    for (int i = threadIdx.x; i < words; i += blockDim.x) sm[i] = in[(blockIdx.x * 977 + i + it * 131) % n];
    __syncthreads();
    for (int i = threadIdx.x; i < words; i += blockDim.x) acc += sm[(i * 7 + it) % words];
    __syncthreads();
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0, reps = argc > 2 ? atoi(argv[2]) : 200;
  cudaStream_t sa, sb;
  cudaStreamCreateWithFlags(&sa, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&sb, cudaStreamNonBlocking);
  // A: the stage-1 GEMM of config 4's 3D parity plan (row-major B, class batch)
  const int M = 96, N = 192, K = 96, batch = 768;
  Gemm a;
  a.M = M; a.N = N; a.K = K; a.batch1 = batch / 2; a.batch2 = 2;
  a.A = dalloc(2LL * M * K, 1); a.a_rs = K; a.a_cs = 1; a.a_b1 = 0; a.a_b2 = (int64_t)M * K;
  a.B = dalloc((int64_t)batch * K * N, 2); a.b_rs = N; a.b_cs = 1; a.b_b1 = 2LL * K * N; a.b_b2 = (int64_t)K * N;
  double* Ca = dalloc((int64_t)batch * M * N, 3);
  a.C = Ca; a.c_rs = N; a.c_cs = 1; a.c_b1 = 2LL * M * N; a.c_b2 = (int64_t)M * N;
  // B: something else on the other stream
  Gemm b;
  if (mode == 0) {  // TMA-ineligible (odd leading dimension of A): cp.async kernel
    b.M = 192; b.N = 192; b.K = 191; b.batch1 = 8;
    b.A = dalloc(8LL * 192 * 191, 4); b.a_rs = 191; b.a_cs = 1; b.a_b1 = 192LL * 191;
    b.B = dalloc(8LL * 191 * 192, 5); b.b_rs = 192; b.b_cs = 1; b.b_b1 = 191LL * 192;
  } else {          // another TMA GEMM (column-major B)
    b.M = 192; b.N = 192; b.K = 192; b.batch1 = 8;
    b.A = dalloc(8LL * 192 * 192, 4); b.a_rs = 192; b.a_cs = 1; b.a_b1 = 192LL * 192;
    b.B = dalloc(8LL * 192 * 192, 5); b.b_rs = 1; b.b_cs = 192; b.b_b1 = 192LL * 192;
  }
  b.C = dalloc(8LL * 192 * 192, 6); b.c_rs = 192; b.c_cs = 1; b.c_b1 = 192LL * 192;
  const int64_t csz = (int64_t)batch * M * N;
  std::vector<double> first(csz), cur(csz);
  if (!try_tma_gemm(a, sa)) { printf("A not taken by the TMA path\n"); return 1; }
  cudaStreamSynchronize(sa);
  cudaMemcpy(first.data(), Ca, csz * 8, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int r = 0; r < reps; r++) {
    cudaMemsetAsync(Ca, 0, csz * 8, sa);
    for (int q = 0; q < 6; q++) {
      if (mode == 3) dummy_smem_kernel<<<288, 128, 38912, sb>>>(b.A, b.C, 8 * 192 * 191);
      else if (mode != 2) run_gemm(b, sb);
      if (q == 2) try_tma_gemm(a, sa);
    }
    cudaStreamSynchronize(sa);
    cudaStreamSynchronize(sb);
    cudaMemcpy(cur.data(), Ca, csz * 8, cudaMemcpyDeviceToHost);
    if (memcmp(cur.data(), first.data(), csz * 8) != 0) {
      int64_t nb = 0, fi = -1;
      for (int64_t i = 0; i < csz; i++)
        if (cur[i] != first[i]) { nb++; if (fi < 0) fi = i; }
      if (bad < 5) printf("rep %d: %lld entries differ, first at batch %lld row %lld col %lld\n", r, (long long)nb,
                          (long long)(fi / (M * N)), (long long)(fi % (M * N) / N), (long long)(fi % N));
      bad++;
    }
  }
  printf("mode %d: %d of %d repetitions differ from the solitary result\n", mode, bad, reps);
  return 0;
}
