// One pass over a 2D block of X for every thin coupling that reads it
// (DESIGN.md §4.2): the Gram blocks that map the PDE block onto a block with a
// single site in one dimension (Eq. 20 with a 1 x n'_i factor) start with a
// point/cell functional of the whole PDE-shaped vector —
//   column type (one output time site, IC-like):  s_c[k1] = sum_k0 wc_c[k0] X[k0][k1]
//   row type (one output space site, BC-like):    t_q[k0] = sum_k1 X[k0][k1] wr_q[k1]
// — each a full read of X when run as its own few-row / few-column GEMM.  Here
// all of them (up to 4 of each type) are evaluated from a single read, and the
// results land in the layout the second contraction of each pair's KronSum
// expects (KronSum::apply with `stage0`).  Sums are accumulated in a fixed
// order (deterministic): rows inside a warp's lane, 8 warps and row tiles in
// index order.
#include "problem.h"

namespace gpfvm {

namespace {
constexpr int FP_TR = 32;      // rows per block tile
constexpr int FP_WARPS = 8;    // warps per block; each owns 64 columns of a 512-column chunk
constexpr int FP_CHUNK = FP_WARPS * 64;

struct FuncArgs {
  int n0, n1, R, NC, NR, tiles;
  const double* wc;   // [4][n0]
  const double* wr;   // [4][n1]
  double* colpart;    // [R][tiles][4][n1]
  double* rout[4];    // row outputs: rout[q] + r * r_rs[q] + k0 * r_ks[q]
  int64_t r_rs[4], r_ks[4];
};

// 16 values per lane (4 rows x 4 functionals) summed over the 32 lanes with a
// halving butterfly (8 + 4 + 2 + 1 + 1 exchanges); afterwards lane l holds the
// total of value index l >> 1.
__device__ __forceinline__ double reduce16(double (&v)[16], int lane) {
#pragma unroll
  for (int k = 0; k < 8; k++) {
    const bool up = lane & 16;
    const double send = up ? v[k] : v[k + 8], keep = up ? v[k + 8] : v[k];
    v[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int k = 0; k < 4; k++) {
    const bool up = lane & 8;
    const double send = up ? v[k] : v[k + 4], keep = up ? v[k + 4] : v[k];
    v[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
#pragma unroll
  for (int k = 0; k < 2; k++) {
    const bool up = lane & 4;
    const double send = up ? v[k] : v[k + 2], keep = up ? v[k + 2] : v[k];
    v[k] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  {
    const bool up = lane & 2;
    const double send = up ? v[0] : v[1], keep = up ? v[1] : v[0];
    v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
  }
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}

// grid (tiles, R), block 256.  Block (tile, r) reads rows [tile*32, tile*32+32)
// of X_r; warp w owns columns [64 w, 64 w + 64) of each 512-column chunk, one
// double2 per lane.
__global__ void __launch_bounds__(FP_WARPS * 32)
    func_pass_kernel(const double* __restrict__ x, int64_t ldx, FuncArgs a) {
  __shared__ double rowpart[FP_TR][4][FP_WARPS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x, r = blockIdx.y;
  const int k00 = tile * FP_TR;
  const double* xr = x + (int64_t)r * ldx;
  for (int i = threadIdx.x; i < FP_TR * 4 * FP_WARPS; i += blockDim.x) (&rowpart[0][0][0])[i] = 0.0;
  __syncthreads();
  for (int c0 = 0; c0 < a.n1; c0 += FP_CHUNK) {
    const int col = c0 + warp * 64 + 2 * lane;
    const bool in = col < a.n1;  // n1 even: col + 1 < n1 as well
    double2 wr[4];
#pragma unroll
    for (int q = 0; q < 4; q++)
      wr[q] = (in && q < a.NR) ? *reinterpret_cast<const double2*>(a.wr + (int64_t)q * a.n1 + col) : make_double2(0.0, 0.0);
    double2 cacc[4];
#pragma unroll
    for (int c = 0; c < 4; c++) cacc[c] = make_double2(0.0, 0.0);
    for (int g = 0; g < FP_TR; g += 4) {
      double v[16];
      double2 xv[4];
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int k0 = k00 + g + u;
        xv[u] = (in && k0 < a.n0) ? *reinterpret_cast<const double2*>(xr + (int64_t)k0 * a.n1 + col) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int k0 = k00 + g + u;
#pragma unroll
        for (int q = 0; q < 4; q++) v[u * 4 + q] = fma(xv[u].x, wr[q].x, xv[u].y * wr[q].y);
#pragma unroll
        for (int c = 0; c < 4; c++) {
          if (c < a.NC) {
            const double w = k0 < a.n0 ? a.wc[(int64_t)c * a.n0 + k0] : 0.0;
            cacc[c].x = fma(w, xv[u].x, cacc[c].x);
            cacc[c].y = fma(w, xv[u].y, cacc[c].y);
          }
        }
      }
      if (a.NR > 0) {
        const double tot = reduce16(v, lane);
        if (!(lane & 1)) {
          const int idx = lane >> 1;  // (row u, functional q) = (idx >> 2, idx & 3)
          rowpart[g + (idx >> 2)][idx & 3][warp] += tot;
        }
      }
    }
    if (in) {
#pragma unroll
      for (int c = 0; c < 4; c++)
        if (c < a.NC)
          *reinterpret_cast<double2*>(a.colpart + (((int64_t)r * a.tiles + tile) * 4 + c) * a.n1 + col) = cacc[c];
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < FP_TR * 4; i += blockDim.x) {
    const int u = i >> 2, q = i & 3, k0 = k00 + u;
    if (q < a.NR && k0 < a.n0) {
      double sum = 0.0;
#pragma unroll
      for (int w = 0; w < FP_WARPS; w++) sum += rowpart[u][q][w];
      a.rout[q][(int64_t)r * a.r_rs[q] + (int64_t)k0 * a.r_ks[q]] = sum;
    }
  }
}

struct ColOut {
  double* out[4];   // out[c] + r * rs[c] + k1
  int64_t rs[4];
};
// column sums: the row-tile partials in tile order
__global__ void func_colsum_kernel(const double* __restrict__ colpart, ColOut o, int R, int tiles, int NC, int n1) {
  const int64_t tot = (int64_t)R * NC * n1;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int k1 = (int)(e % n1);
    const int c = (int)((e / n1) % NC), r = (int)(e / ((int64_t)n1 * NC));
    double sum = 0.0;
    for (int t = 0; t < tiles; t++) sum += colpart[(((int64_t)r * tiles + t) * 4 + c) * n1 + k1];
    o.out[c][(int64_t)r * o.rs[c] + k1] = sum;
  }
}
}  // namespace

void FusedFunc::ensure(int R) {
  zbuf.ensure((size_t)std::max<int64_t>(1, zper * R));
  colpart.ensure((size_t)std::max<int64_t>(1, (int64_t)R * tiles() * 4 * n1));
}

int FusedFunc::tiles() const { return (n0 + FP_TR - 1) / FP_TR; }

void FusedFunc::run(const double* xJ, int64_t ldx, int R, cudaStream_t s) const {
  FuncArgs a;
  a.n0 = n0; a.n1 = n1; a.R = R; a.NC = NC; a.NR = NR; a.tiles = tiles();
  a.wc = wc.ptr; a.wr = wr.ptr; a.colpart = colpart.ptr;
  ColOut co;
  for (int q = 0; q < 4; q++) {
    a.rout[q] = nullptr; a.r_rs[q] = a.r_ks[q] = 0;
    co.out[q] = nullptr; co.rs[q] = 0;
  }
  for (const Out& o : outs) {
    // pair buffers are laid out for R vectors: zbuf + off * R
    double* base = zbuf.ptr + o.off * R;
    for (int p = 0; p < o.P; p++) {
      if (o.type == 0) {  // Z_r[p][k1]
        co.out[o.first + p] = base + (int64_t)p * n1;
        co.rs[o.first + p] = (int64_t)o.P * n1;
      } else {            // Z_r[k0][p]
        a.rout[o.first + p] = base + p;
        a.r_rs[o.first + p] = (int64_t)n0 * o.P;
        a.r_ks[o.first + p] = o.P;
      }
    }
  }
  func_pass_kernel<<<dim3((unsigned)a.tiles, (unsigned)R), FP_WARPS * 32, 0, s>>>(xJ, ldx, a);
  count_launch();
  if (NC > 0) {
    const int64_t tot = (int64_t)R * NC * n1;
    func_colsum_kernel<<<(unsigned)std::min<int64_t>((tot + 255) / 256, 148 * 8), 256, 0, s>>>(colpart.ptr, co, R,
                                                                                               a.tiles, NC, n1);
    count_launch();
  }
  check_launch("FusedFunc::run");
}

const double* FusedFunc::stage0_of(int pair, int R) const {
  for (const Out& o : outs)
    if (o.pair == pair) return zbuf.ptr + o.off * R;
  return nullptr;
}

// Collect the thin pairs (I, J) of every 2D input block J into one pass.
void build_fused_func(gpfvm_problem* p, MatvecPlan& pl, cudaStream_t s) {
  pl.fused.clear();
  static const bool off = getenv("GPFVM_NO_FUNCPASS") != nullptr;
  if (off || p->ndim != 2) return;
  const int nb = (int)p->blocks.size();
  for (int J = 0; J < nb; J++) {
    const int n0 = p->blocks[J].shape[0], n1 = p->blocks[J].shape[1];
    if (n0 < 2 || n1 < 2 || (n1 & 1) || (p->blocks[J].offset & 1)) continue;
    FusedFunc ff;
    ff.J = J; ff.n0 = n0; ff.n1 = n1;
    std::vector<int> cand;
    for (size_t k = 0; k < pl.pairs.size(); k++) {
      const PairOp& op = pl.pairs[k];
      const KronSum& ks = op.ks;
      if (op.J != J || op.I == J || op.lowrank || ks.par || ks.d != 2 || ks.P == 0) continue;
      const bool col = ks.nout[0] == 1 && !ks.rev, row = ks.nout[1] == 1 && ks.rev;
      if (col && !row && ff.NC + ks.P <= 4) {
        ff.outs.push_back({(int)k, 0, ks.P, ff.NC, ff.zper});
        ff.NC += ks.P;
        ff.zper += (int64_t)ks.P * n1;
      } else if (row && !col && ff.NR + ks.P <= 4) {
        ff.outs.push_back({(int)k, 1, ks.P, ff.NR, ff.zper});
        ff.NR += ks.P;
        ff.zper += (int64_t)ks.P * n0;
      }
    }
    if (ff.outs.size() < 2) continue;  // a single functional is already one read
    ff.wc.ensure((size_t)4 * n0);
    ff.wr.ensure((size_t)4 * n1);
    fill(ff.wc.ptr, 0.0, 4 * (int64_t)n0, s);
    fill(ff.wr.ptr, 0.0, 4 * (int64_t)n1, s);
    GPFVM_CUDA(cudaEventCreateWithFlags(&ff.ev, cudaEventDisableTiming));
    pl.fused.push_back(std::move(ff));
  }
  pl.fused_of.assign(pl.pairs.size(), -1);
  for (size_t f = 0; f < pl.fused.size(); f++)
    for (const auto& o : pl.fused[f].outs) pl.fused_of[o.pair] = (int)f;
  refresh_fused_func(pl, s);
}

// The functional weights are the pairs' stage-0 factors (coefficients folded
// in): copied again whenever the factors are re-assembled.
void refresh_fused_func(MatvecPlan& pl, cudaStream_t s) {
  for (auto& ff : pl.fused)
    for (const auto& o : ff.outs) {
      const KronSum& ks = pl.pairs[o.pair].ks;
      // the plan of a thin pair is fixed by its shapes (re-assembly keeps it)
      GPFVM_CHECK(ks.P == o.P && (o.type == 0 ? !ks.rev : ks.rev), GPFVM_ERR_STATE, "fused functional plan changed");
      // column type (forward order): stk[0] = c_p F0^p rows (P x n0); row type
      // (reverse order): stk[1] = c_p F1^p rows (P x n1)
      if (o.type == 0)
        GPFVM_CUDA(cudaMemcpyAsync(ff.wc.ptr + (int64_t)o.first * ff.n0, ks.stk[0].ptr, sizeof(double) * o.P * ff.n0,
                                   cudaMemcpyDeviceToDevice, s));
      else
        GPFVM_CUDA(cudaMemcpyAsync(ff.wr.ptr + (int64_t)o.first * ff.n1, ks.stk[1].ptr, sizeof(double) * o.P * ff.n1,
                                   cudaMemcpyDeviceToDevice, s));
    }
}

}  // namespace gpfvm
