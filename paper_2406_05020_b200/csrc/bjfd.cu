// Block-Jacobi fast-diagonalisation preconditioner for
// problems outside the exact 2D two-term case (3D wave / advection-diffusion,
// multi-output shallow water): for every observation block J
//   Q_i  = generalised eigenvectors of (F_i^{lo,lo}, F_i^{hi,hi})  per dimension
//          (lowest / highest derivative order of the block's terms in dim i;
//           orthonormal eigenvectors of F_i^{lo,lo} if both coincide)
//   D    = sum_(tau,tau') c c' (x)_i diag(Q_i^T F_i^{(tau,tau')} Q_i) + noise (x)_i diag(Q_i^T Q_i)
//   P_J^{-1} = ((x)_i Q_i) D^{-1} ((x)_i Q_i)^T
// i.e. the block's Gram with every Kronecker term replaced by its diagonal in
// the common basis (exact for the heat block, R6); couplings between blocks
// are left to the Krylov iteration.
#include "problem.h"

namespace gpfvm {

namespace {
unsigned gsz(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 4096)); }

__global__ void eye2(double* A, int n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < (int64_t)n * n) A[i] = (i / n == i % n) ? 1.0 : 0.0;
}
// d[k] = sum_a Q[a][k] T[a][k]
__global__ void coldot_kernel(const double* __restrict__ Q, const double* __restrict__ T, int n, double* d) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  double s = 0.0;
  for (int a = 0; a < n; a++) s = fma(Q[(int64_t)a * n + k], T[(int64_t)a * n + k], s);
  d[k] = s;
}
// D[idx] += c * prod_i d_i[idx_i]   (row-major over shape, up to 4 dims)
__global__ void outer_acc_kernel(double* D, int4 shape, const double* d0, const double* d1, const double* d2,
                                 const double* d3, double c, int64_t total) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i;
    int i3 = (int)(r % shape.w); r /= shape.w;
    int i2 = (int)(r % shape.z); r /= shape.z;
    int i1 = (int)(r % shape.y); r /= shape.y;
    int i0 = (int)r;
    D[i] += c * d0[i0] * d1[i1] * d2[i2] * d3[i3];
  }
}
__global__ void recip_clamp_kernel(double* D, int64_t n, double floor_) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    D[i] = 1.0 / fmax(D[i], floor_);
}
__global__ void ones_kernel(double* x, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = 1.0;
}
__global__ void maxabs_kernel(const double* x, int64_t n, unsigned long long* out) {
  double m = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, fabs(x[i]));
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}
__global__ void vmul2(double* x, const double* __restrict__ d, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] *= d[i];
}
}  // namespace

void build_block_fd(gpfvm_problem* p, int J, BlockFD& bf, cudaStream_t s, PencilCache* cache) {
  const BlockInt& B = p->blocks[J];
  const int d = p->ndim;
  bf.J = J;
  bf.d = d;
  for (int i = 0; i < GPFVM_MAX_DIMS; i++) bf.shape[i] = (i < d) ? B.shape[i] : 1;
  const int out = B.terms[0].output;
  DevBuf I;
  for (int i = 0; i < d; i++) {
    const int n = B.shape[i];
    bf.Q[i].ensure((size_t)n * n);
    bf.Qt[i].ensure((size_t)n * n);
    int lo = 1 << 30, hi = -1;
    for (const auto& t : B.terms)
      if (t.output == out) {
        lo = std::min(lo, t.order[i]);
        hi = std::max(hi, t.order[i]);
      }
    if (n == 1) {
      eye2<<<1, 32, 0, s>>>(bf.Q[i].ptr, 1);
      count_launch();
    } else {
      const int fa = get_factor(p, out, i, J, lo, J, lo), fb = get_factor(p, out, i, J, hi, J, hi);
      const Factor& A = p->factors[fa];
      const Factor& Bm = p->factors[fb];
      GPFVM_CHECK(A.data.ptr && Bm.data.ptr, GPFVM_ERR_STATE, "block FD: diagonal factors not assembled");
      const Sites& st = B.sites[i];
      const PencilKey key{out, i, lo, lo == hi ? -1 : hi, st.kind, st.lo, st.hi};
      DevBuf w;
      w.ensure(n);
      if (cache && cache->count(key)) {
        // same pencil as an earlier block (e.g. the time factors of the faces)
        GPFVM_CUDA(cudaMemcpyAsync(bf.Q[i].ptr, cache->at(key), sizeof(double) * n * n, cudaMemcpyDeviceToDevice, s));
      } else if (lo == hi) {
        I.ensure((size_t)n * n);
        eye2<<<gsz((int64_t)n * n), 256, 0, s>>>(I.ptr, n);
        count_launch();
        sygv(A.data.ptr, I.ptr, n, bf.Q[i].ptr, w.ptr, s);
      } else {
        sygv(A.data.ptr, Bm.data.ptr, n, bf.Q[i].ptr, w.ptr, s);
      }
      if (cache && !cache->count(key)) (*cache)[key] = bf.Q[i].ptr;
    }
    transpose(bf.Q[i].ptr, bf.Qt[i].ptr, n, n, s);
  }
  // D = sum over the block's diagonal Kronecker terms of the per-dim diagonals in the Q basis
  bf.Dinv.ensure((size_t)B.size);
  fill(bf.Dinv.ptr, 0.0, B.size, s);
  std::map<int, DevBuf> diag;  // factor id -> diag(Q^T F Q)
  DevBuf T, ones;
  ones.ensure(1);
  ones_kernel<<<1, 32, 0, s>>>(ones.ptr, 1);
  count_launch();
  auto diag_of = [&](int fid, int i) -> const double* {
    auto it = diag.find(fid);
    if (it != diag.end()) return it->second.ptr;
    const int n = B.shape[i];
    DevBuf& dv = diag[fid];
    dv.ensure(n);
    T.ensure((size_t)n * n);
    Gemm g;  // T = F Q
    g.M = n; g.N = n; g.K = n;
    g.A = p->factors[fid].data.ptr; g.a_rs = n; g.a_cs = 1;
    g.B = bf.Q[i].ptr; g.b_rs = n; g.b_cs = 1;
    g.C = T.ptr; g.c_rs = n; g.c_cs = 1;
    run_gemm(g, s);
    coldot_kernel<<<gsz(n), 256, 0, s>>>(bf.Q[i].ptr, T.ptr, n, dv.ptr);
    count_launch();
    return dv.ptr;
  };
  const int4 shp = make_int4(bf.shape[0], bf.shape[1], bf.shape[2], bf.shape[3]);
  for (const auto& t : p->terms) {
    if (t.I != J || t.J != J) continue;
    const double* dv[4] = {ones.ptr, ones.ptr, ones.ptr, ones.ptr};
    for (int i = 0; i < d; i++) dv[i] = diag_of(t.fid[i], i);
    outer_acc_kernel<<<gsz(B.size), 256, 0, s>>>(bf.Dinv.ptr, shp, dv[0], dv[1], dv[2], dv[3], t.coef, B.size);
    count_launch();
  }
  if (B.noise > 0.0) {
    // noise * (x)_i diag(Q_i^T Q_i): column sums of squares
    std::vector<DevBuf> qq(d);
    const double* dv[4] = {ones.ptr, ones.ptr, ones.ptr, ones.ptr};
    for (int i = 0; i < d; i++) {
      const int n = B.shape[i];
      qq[i].ensure(n);
      coldot_kernel<<<gsz(n), 256, 0, s>>>(bf.Q[i].ptr, bf.Q[i].ptr, n, qq[i].ptr);
      count_launch();
      dv[i] = qq[i].ptr;
    }
    outer_acc_kernel<<<gsz(B.size), 256, 0, s>>>(bf.Dinv.ptr, shp, dv[0], dv[1], dv[2], dv[3], B.noise, B.size);
    count_launch();
    GPFVM_CUDA(cudaStreamSynchronize(s));
  }
  // D^{-1}, clamping non-positive diagonal estimates at 1e-14 max|D|
  DevBuf mx;
  mx.ensure(1);
  GPFVM_CUDA(cudaMemsetAsync(mx.ptr, 0, sizeof(double), s));
  maxabs_kernel<<<gsz(B.size), 256, 0, s>>>(bf.Dinv.ptr, B.size, reinterpret_cast<unsigned long long*>(mx.ptr));
  count_launch();
  double hmax = 0.0;
  GPFVM_CUDA(cudaMemcpyAsync(&hmax, mx.ptr, sizeof(double), cudaMemcpyDeviceToHost, s));
  GPFVM_CUDA(cudaStreamSynchronize(s));
  recip_clamp_kernel<<<gsz(B.size), 256, 0, s>>>(bf.Dinv.ptr, B.size, 1e-14 * hmax);
  count_launch();
  // forward (Q^T) and backward (Q) single-term Kronecker operators
  std::vector<std::vector<const double*>> ft(1), fb(1);
  for (int i = 0; i < d; i++) {
    ft[0].push_back(bf.Qt[i].ptr);
    fb[0].push_back(bf.Q[i].ptr);
  }
  bf.fwd.build(d, B.shape, B.shape, {1.0}, ft, s);
  bf.bwd.build(d, B.shape, B.shape, {1.0}, fb, s);
  const int64_t ws = std::max<int64_t>(1, std::max(bf.fwd.workspace_per_rhs(), bf.bwd.workspace_per_rhs()));
  bf.w0.ensure(ws);
  bf.w1.ensure(ws);
  bf.tmp.ensure(B.size);
  check_launch("build_block_fd");
  GPFVM_CUDA(cudaStreamSynchronize(s));
}

__global__ void vmul_many(double* x, int64_t ldx, const double* __restrict__ d, int64_t n) {
  double* xr = x + blockIdx.y * ldx;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    xr[i] *= d[i];
}

// z_J = Q D^{-1} Q^T r_J for R vectors (strides ldr, ldz); tmp: R * n doubles,
// w0/w1: R * workspace doubles each (caller-owned)
void apply_block_fd_many(const BlockFD& bf, const double* r, int64_t ldr, double* z, int64_t ldz, int64_t n, int R,
                         double* tmp, double* w0, double* w1, cudaStream_t s) {
  bf.fwd.apply(r, ldr, tmp, n, R, 0.0, w0, w1, s);
  vmul_many<<<dim3(gsz(n), R), 256, 0, s>>>(tmp, n, bf.Dinv.ptr, n);
  count_launch();
  bf.bwd.apply(tmp, n, z, ldz, R, 0.0, w0, w1, s);
}

// z_J = Q D^{-1} Q^T r_J
void apply_block_fd(const BlockFD& bf, const double* r, double* z, int64_t n, cudaStream_t s) {
  bf.fwd.apply(r, n, bf.tmp.ptr, n, 1, 0.0, bf.w0.ptr, bf.w1.ptr, s);
  vmul2<<<gsz(n), 256, 0, s>>>(bf.tmp.ptr, bf.Dinv.ptr, n);
  count_launch();
  bf.bwd.apply(bf.tmp.ptr, n, z, n, 1, 0.0, bf.w0.ptr, bf.w1.ptr, s);
}

}  // namespace gpfvm
