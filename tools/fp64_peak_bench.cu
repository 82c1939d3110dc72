#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0+1, x2 = x0+2, x3 = x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < 8; u++) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0+x1+x2+x3+x4+x5+x6+x7;
}
__global__ void dmma884_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x*1e-4;
  double c[8][2];
  for (int i = 0; i < 8; i++) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0; for (int i = 0; i < 8; i++) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void dmma16816_kernel(double* out, int iters) {
  double a[8], b[4];
  for (int i = 0; i < 8; i++) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 4; i++) b[i] = 1.0 - threadIdx.x*1e-4 + i;
  double c[4][4];
  for (int i = 0; i < 4; i++) for (int j = 0; j < 4; j++) c[i][j] = 0;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 4; i++) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
        : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
        : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
          "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0; for (int i = 0; i < 4; i++) for (int j = 0; j < 4; j++) s += c[i][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void dmma1688_kernel(double* out, int iters) {
  double a[4], b[2];
  for (int i = 0; i < 4; i++) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 2; i++) b[i] = 1.0 - threadIdx.x*1e-4 + i;
  double c[4][4];
  for (int i = 0; i < 4; i++) for (int j = 0; j < 4; j++) c[i][j] = 0;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 4; i++) {
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
        : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
    }
  }
  double s = 0; for (int i = 0; i < 4; i++) for (int j = 0; j < 4; j++) s += c[i][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void copy_kernel(const double2* __restrict__ in, double2* __restrict__ out, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) out[i] = in[i];
}
int main() {
  double* out; cudaMalloc(&out, 148*32*1024*sizeof(double));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int rep = 0; rep < 2; rep++) {
  { int iters = 4096, blocks = sms*8, threads = 256;
    dfma_kernel<<<blocks, threads>>>(out, 16, 1.0000001, 1e-9);
    cudaEventRecord(e0); dfma_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 64 * iters * (double)blocks * threads;
    printf("DFMA: %.2f TFLOP/s (%.3f ms)\n", flops / ms / 1e9, ms); }
  for (int tpb : {128, 256, 512}) { int iters = 4096, blocks = sms*4;
    dmma884_kernel<<<blocks, tpb>>>(out, 16);
    cudaEventRecord(e0); dmma884_kernel<<<blocks, tpb>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8*8*4 * 8 * iters * (double)blocks * (tpb/32);
    printf("DMMA m8n8k4 tpb=%d: %.2f TFLOP/s (%.3f ms)\n", tpb, flops / ms / 1e9, ms); }
  for (int tpb : {128, 256, 512}) { int iters = 1024, blocks = sms*4;
    dmma16816_kernel<<<blocks, tpb>>>(out, 16);
    cudaEventRecord(e0); dmma16816_kernel<<<blocks, tpb>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16*8*16 * 4 * iters * (double)blocks * (tpb/32);
    printf("DMMA m16n8k16 tpb=%d: %.2f TFLOP/s (%.3f ms)\n", tpb, flops / ms / 1e9, ms); }
  for (int tpb : {128, 256, 512}) { int iters = 2048, blocks = sms*4;
    dmma1688_kernel<<<blocks, tpb>>>(out, 16);
    cudaEventRecord(e0); dmma1688_kernel<<<blocks, tpb>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16*8*8 * 4 * iters * (double)blocks * (tpb/32);
    printf("DMMA m16n8k8 tpb=%d: %.2f TFLOP/s (%.3f ms)\n", tpb, flops / ms / 1e9, ms); }
  { size_t n = (size_t)1 << 28; double2 *a, *b; cudaMalloc(&a, n*16); cudaMalloc(&b, n*16); cudaMemset(a, 0, n*16);
    copy_kernel<<<sms*8, 512>>>(a, b, n);
    float best = 1e9; for (int i = 0; i < 5; i++) { cudaEventRecord(e0); copy_kernel<<<sms*8, 512>>>(a, b, n); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
    printf("copy: %.1f GB/s\n", 2.0*n*16/best/1e6); cudaFree(a); cudaFree(b); }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
