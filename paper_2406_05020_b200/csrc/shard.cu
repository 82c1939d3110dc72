// Time-mode sharded GP-FVM operators (north_star multi-GPU row).
//
// Every observation block whose dimension 0 is the common time axis (n0
// sites) is split into W contiguous time slabs, rank r owning sites
// [r n0 / W, (r+1) n0 / W); blocks with a single time site (IC planes) live on
// rank 0.  A Kronecker-sum operator (the Gram of Eq. 20, or the block-Jacobi
// FD transforms) is applied as
//   begin : for every output block I and every distinct time factor q of I,
//           Z_q = sum_{J, p in q} c_p (I_t (x) F1_p (x) ...) x_J      (local rows,
//           spatial Kronecker products; terms sharing a time factor are summed
//           before any communication: (Q + 1) N bytes per matvec instead of
//           (P + 1) N), packed per destination spatial chunk;
//   [caller: all-to-all #1]
//   mid   : per time-extended output I, one K-concatenated GEMM over all
//           time rows of every group:  Y_I[:, chunk] = [F0_q1 | F0_q2 | ...] Z,
//           packed per owner of the output time rows; single-time outputs
//           (IC planes) are contracted locally over the owned time rows and
//           their partial sums shipped to rank 0;
//   [caller: all-to-all #2]
//   end   : y_local = noise x_local + the received rows (rank 0 adds the
//           partial sums of the single-time outputs in rank order).
// The library owns every arithmetic step; the caller (dist.py) only moves the
// buffers with NCCL all_to_all_single and all_reduces the IterGP scalars.
#include <algorithm>
#include <map>
#include <memory>
#include <vector>

#include "problem.h"

namespace gpfvm {

namespace {

struct CopyDesc {
  int64_t src_off, dst_off;
  int64_t rows, cols, src_ld, dst_ld;
};

// dst[desc] (+)= src[desc], one descriptor per blockIdx.y; descriptors of one
// launch write disjoint destinations
__global__ void batched_copy_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                    const CopyDesc* __restrict__ descs, int accumulate) {
  const CopyDesc c = descs[blockIdx.y];
  const int64_t total = c.rows * c.cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / c.cols, k = i - r * c.cols;
    const double v = src[c.src_off + r * c.src_ld + k];
    double* o = dst + c.dst_off + r * c.dst_ld + k;
    *o = accumulate ? *o + v : v;
  }
}

__global__ void shard_noise_kernel(double* __restrict__ y, const double* __restrict__ x,
                                   const double* __restrict__ noise, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = noise[i] * x[i];
}

__global__ void shard_vmul_kernel(double* __restrict__ x, const double* __restrict__ d, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] *= d[i];
}

unsigned gsz(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 4096)); }

struct DescList {
  std::vector<CopyDesc> h;
  DevBuf d;  // device copy (doubles-sized storage)
  void upload(cudaStream_t s) {
    if (h.empty()) return;
    const size_t bytes = h.size() * sizeof(CopyDesc);
    d.ensure((bytes + 7) / 8);
    GPFVM_CUDA(cudaMemcpyAsync(d.ptr, h.data(), bytes, cudaMemcpyHostToDevice, s));
  }
  void run(const double* src, double* dst, bool acc, cudaStream_t s) const {
    if (h.empty()) return;
    int64_t mx = 1;
    for (const auto& c : h) mx = std::max(mx, c.rows * c.cols);
    const dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>((mx + 255) / 256, 1024)), (unsigned)h.size());
    batched_copy_kernel<<<grid, 256, 0, s>>>(src, dst, reinterpret_cast<const CopyDesc*>(d.ptr), acc ? 1 : 0);
    count_launch();
    check_launch("batched_copy_kernel");
  }
};

}  // namespace

// One term of a sharded Kronecker-sum operator: coef (x)_i f[i] from block J
// to block I; tkey identifies the value of the time factor f[0] (terms of the
// same output with equal tkey are summed before the exchange).
struct ShardTermIn {
  int I = 0, J = 0;
  double coef = 0.0;
  const double* f[GPFVM_MAX_DIMS] = {nullptr, nullptr, nullptr, nullptr};
  int sg[GPFVM_MAX_DIMS] = {0, 0, 0, 0};  // reflection parity of each factor (Factor::psign; 0: none)
  int64_t tkey = 0;
};

struct ShardLayout {
  int rank = 0, world = 1, d = 0, n0 = 1, nb = 0;
  std::vector<int> shape0;           // time extent per block
  std::vector<int64_t> spatial;      // spatial size per block
  std::vector<int64_t> loc_off;      // offset of the block in the local vector
  int64_t local_n = 0;
  bool ext(int J) const { return shape0[J] > 1; }
  int t_lo(int r) const { return (int)((int64_t)r * n0 / world); }
  int rows(int J, int r) const { return ext(J) ? t_lo(r + 1) - t_lo(r) : (r == 0 ? 1 : 0); }
  int row0(int J, int r) const { return ext(J) ? t_lo(r) : 0; }
  int64_t c_lo(int I, int r) const { return spatial[I] * r / world; }
  int64_t chunk(int I, int r) const { return c_lo(I, r + 1) - c_lo(I, r); }
};

ShardLayout make_layout(const gpfvm_problem* p, int rank, int world) {
  ShardLayout L;
  L.rank = rank;
  L.world = world;
  L.d = p->ndim;
  L.nb = (int)p->blocks.size();
  GPFVM_CHECK(L.d >= 2, GPFVM_ERR_UNSUPPORTED, "sharding needs >= 2 dimensions (dimension 0 is split)");
  for (const auto& B : p->blocks) L.n0 = std::max(L.n0, B.shape[0]);
  for (const auto& B : p->blocks) {
    GPFVM_CHECK(B.shape[0] == 1 || B.shape[0] == L.n0, GPFVM_ERR_UNSUPPORTED,
                "sharding: every block needs either the common time extent or a single time site");
    L.shape0.push_back(B.shape[0]);
    L.spatial.push_back(B.size / B.shape[0]);
  }
  GPFVM_CHECK(world >= 1 && rank >= 0 && rank < world && (L.n0 == 1 || world <= L.n0), GPFVM_ERR_INVALID,
              "bad rank / world size (world must not exceed the time extent)");
  for (int J = 0; J < L.nb; J++) {
    L.loc_off.push_back(L.local_n);
    L.local_n += (int64_t)L.rows(J, rank) * L.spatial[J];
  }
  return L;
}

// Sharded Kronecker-sum operator over the block structure (one rank's part).
struct ShardOp {
  ShardLayout L;
  struct Member {
    int J = 0;
    std::vector<double> coefs;                     // terms of the pair (I, J) in this group
    std::vector<std::vector<const double*>> fs;    // their spatial factors (dims 1..d-1)
    std::vector<std::vector<int>> sgn;             // and the factors' reflection parities (KronSum parity split)
    KronSum ks;  // spatial (d-1)-dim Kronecker sum J -> I (coefficients folded)
  };
  struct Group {
    int I = 0, tJ = 0;         // output block, representative input block (time rows)
    const double* F0 = nullptr;  // time factor (n0_I x n0_J), row-major
    int n0I = 1, n0J = 1;
    std::vector<Member> mem;
    int64_t zoff = 0;          // offset of Z_q in Zall ([rows(tJ, me)][S_I])
    int64_t koff = 0;          // column offset of F0 in A_I (time-extended outputs)
  };
  std::vector<Group> groups;
  std::vector<std::vector<int>> by_out;  // group indices per output block
  // time-extended outputs
  std::vector<int64_t> boff, yoff, ldc, Kdim;  // per output block (ext only)
  std::vector<DevBuf> A;                        // [n0 x K_I] per ext output
  std::vector<int64_t> poff;                    // single-time outputs: partial offset in Pall
  DevBuf Zall, Ball, Yall, Pall, w0, w1;
  std::vector<int64_t> send1, recv1, send2, recv2;  // counts per rank
  DescList pack1, unpack1, pack2y, pack2p, unpack2;
  std::vector<DescList> unpack2_single;  // per source rank (rank 0 only): single-time partials, accumulated in rank order

  // host part: groups, buffer offsets, exchange counts and copy descriptors
  void plan(const ShardLayout& lay, const std::vector<ShardTermIn>& terms);
  // device part: spatial Kronecker sums, buffers, A_I, descriptors uploaded
  void materialize(const gpfvm_problem* p, cudaStream_t s);
  void build(const gpfvm_problem* p, const ShardLayout& lay, const std::vector<ShardTermIn>& terms,
             const std::vector<const double*>&, cudaStream_t s) {
    plan(lay, terms);
    materialize(p, s);
  }
  int64_t wsz = 1, zsz = 0, bsz = 0, ysz = 0, psz = 0;
  void begin(const double* x, double* sendbuf, cudaStream_t s);
  void mid(const double* recvbuf, double* sendbuf, cudaStream_t s);
  void end(const double* recvbuf, double* y, cudaStream_t s);
};

void ShardOp::plan(const ShardLayout& lay, const std::vector<ShardTermIn>& terms) {
  L = lay;
  const int W = L.world, me = L.rank, nb = L.nb, d = L.d;
  // ---- groups: (output I, time key), members by input block J ----
  std::map<std::pair<int, int64_t>, int> gid;
  std::map<std::pair<int, int>, std::vector<const ShardTermIn*>> per_member;  // (group, J) -> terms
  for (const auto& t : terms) {
    auto key = std::make_pair(t.I, t.tkey);
    auto it = gid.find(key);
    int g;
    if (it == gid.end()) {
      g = (int)groups.size();
      gid[key] = g;
      Group G;
      G.I = t.I;
      G.tJ = t.J;
      G.F0 = t.f[0];
      G.n0I = L.shape0[t.I];
      G.n0J = L.shape0[t.J];
      groups.push_back(std::move(G));
    } else {
      g = it->second;
      GPFVM_CHECK(L.shape0[t.J] == groups[g].n0J, GPFVM_ERR_STATE, "shard: time key shared by different time extents");
    }
    per_member[{g, t.J}].push_back(&t);
  }
  by_out.assign(nb, {});
  for (int g = 0; g < (int)groups.size(); g++) by_out[groups[g].I].push_back(g);
  for (auto& kv : per_member) {
    Group& G = groups[kv.first.first];
    Member m;
    m.J = kv.first.second;
    for (const ShardTermIn* t : kv.second) {
      m.coefs.push_back(t->coef);
      m.fs.push_back(std::vector<const double*>(t->f + 1, t->f + d));
      m.sgn.push_back(std::vector<int>(t->sg + 1, t->sg + d));
    }
    G.mem.push_back(std::move(m));
  }
  for (auto& G : groups) {
    G.zoff = zsz;
    zsz += (int64_t)L.rows(G.tJ, me) * L.spatial[G.I];
  }
  // ---- time-extended outputs: A_I = [F0_q ...], B / Y buffers (even leading dimension) ----
  boff.assign(nb, 0); yoff.assign(nb, 0); ldc.assign(nb, 0); Kdim.assign(nb, 0); poff.assign(nb, 0);
  for (int I = 0; I < nb; I++) {
    if (by_out[I].empty()) continue;
    if (L.ext(I)) {
      const int64_t ch = L.chunk(I, me);
      ldc[I] = std::max<int64_t>(2, ch + (ch & 1));
      int64_t K = 0;
      for (int g : by_out[I]) {
        groups[g].koff = K;
        K += groups[g].n0J;
      }
      Kdim[I] = K;
      boff[I] = bsz;
      bsz += K * ldc[I];
      yoff[I] = ysz;
      ysz += (int64_t)L.n0 * ldc[I];
    } else {
      poff[I] = psz;
      psz += L.spatial[I];
    }
  }
  // ---- exchange layouts ----
  send1.assign(W, 0); recv1.assign(W, 0); send2.assign(W, 0); recv2.assign(W, 0);
  // exchange 1: [peer][ext I][group q] blocks of rows(q, sender) x chunk(I, receiver)
  int64_t so = 0;
  for (int r = 0; r < W; r++) {
    for (int I = 0; I < nb; I++) {
      if (!L.ext(I)) continue;
      for (int g : by_out[I]) {
        const Group& G = groups[g];
        const int64_t rows = L.rows(G.tJ, me), cols = L.chunk(I, r);
        if (rows * cols > 0) pack1.h.push_back({G.zoff + L.c_lo(I, r), so, rows, cols, L.spatial[I], cols});
        so += rows * cols;
        send1[r] += rows * cols;
      }
    }
  }
  int64_t ro = 0;
  for (int r = 0; r < W; r++) {
    for (int I = 0; I < nb; I++) {
      if (!L.ext(I)) continue;
      for (int g : by_out[I]) {
        const Group& G = groups[g];
        const int64_t rows = L.rows(G.tJ, r), cols = L.chunk(I, me);
        if (rows * cols > 0)
          unpack1.h.push_back({ro, boff[I] + (G.koff + L.row0(G.tJ, r)) * ldc[I], rows, cols, cols, ldc[I]});
        ro += rows * cols;
        recv1[r] += rows * cols;
      }
    }
  }
  // exchange 2: [peer][ext I] rows owned by the peer x my chunk; then (peer 0)
  // the single-time partials
  so = 0;
  for (int r = 0; r < W; r++) {
    for (int I = 0; I < nb; I++) {
      if (by_out[I].empty() || !L.ext(I)) continue;
      const int64_t rows = L.rows(I, r), cols = L.chunk(I, me);
      if (rows * cols > 0) pack2y.h.push_back({yoff[I] + (int64_t)L.row0(I, r) * ldc[I], so, rows, cols, ldc[I], cols});
      so += rows * cols;
      send2[r] += rows * cols;
    }
    if (r == 0)
      for (int I = 0; I < nb; I++) {
        if (by_out[I].empty() || L.ext(I)) continue;
        pack2p.h.push_back({poff[I], so, 1, L.spatial[I], L.spatial[I], L.spatial[I]});
        so += L.spatial[I];
        send2[r] += L.spatial[I];
      }
  }
  ro = 0;
  unpack2_single.clear();
  unpack2_single.resize(W);
  for (int r = 0; r < W; r++) {
    for (int I = 0; I < nb; I++) {
      if (by_out[I].empty() || !L.ext(I)) continue;
      const int64_t rows = L.rows(I, me), cols = L.chunk(I, r);
      if (rows * cols > 0) unpack2.h.push_back({ro, L.loc_off[I] + L.c_lo(I, r), rows, cols, cols, L.spatial[I]});
      ro += rows * cols;
      recv2[r] += rows * cols;
    }
    if (me == 0)
      for (int I = 0; I < nb; I++) {
        if (by_out[I].empty() || L.ext(I)) continue;
        unpack2_single[r].h.push_back({ro, L.loc_off[I], 1, L.spatial[I], L.spatial[I], L.spatial[I]});
        ro += L.spatial[I];
        recv2[r] += L.spatial[I];
      }
  }
}

void ShardOp::materialize(const gpfvm_problem* p, cudaStream_t s) {
  const int me = L.rank, nb = L.nb, d = L.d;
  for (auto& G : groups)
    for (auto& m : G.mem) {
      m.ks.build(d - 1, p->blocks[m.J].shape + 1, p->blocks[G.I].shape + 1, m.coefs, m.fs, s, &m.sgn);
      wsz = std::max<int64_t>(wsz, m.ks.workspace_per_rhs() * std::max(1, L.rows(m.J, me)));
    }
  Zall.ensure((size_t)std::max<int64_t>(1, zsz));
  w0.ensure((size_t)wsz);
  w1.ensure((size_t)wsz);
  A.resize(nb);
  for (int I = 0; I < nb; I++) {
    if (by_out[I].empty() || !L.ext(I)) continue;
    A[I].ensure((size_t)L.n0 * Kdim[I]);
    for (int g : by_out[I])
      GPFVM_CUDA(cudaMemcpy2DAsync(A[I].ptr + groups[g].koff, Kdim[I] * sizeof(double), groups[g].F0,
                                   groups[g].n0J * sizeof(double), groups[g].n0J * sizeof(double), L.n0,
                                   cudaMemcpyDeviceToDevice, s));
  }
  Ball.ensure((size_t)std::max<int64_t>(1, bsz));
  Yall.ensure((size_t)std::max<int64_t>(1, ysz));
  Pall.ensure((size_t)std::max<int64_t>(1, psz));
  pack1.upload(s);
  unpack1.upload(s);
  pack2y.upload(s);
  pack2p.upload(s);
  unpack2.upload(s);
  for (auto& u : unpack2_single) u.upload(s);
  check_launch("ShardOp::materialize");
  GPFVM_CUDA(cudaStreamSynchronize(s));
}

void ShardOp::begin(const double* x, double* sendbuf, cudaStream_t s) {
  const int me = L.rank;
  for (auto& G : groups) {
    const int64_t rows = L.rows(G.tJ, me);
    if (rows == 0) continue;
    bool first = true;
    for (const auto& m : G.mem) {
      m.ks.apply(x + L.loc_off[m.J], L.spatial[m.J], Zall.ptr + G.zoff, L.spatial[G.I], (int)rows, first ? 0.0 : 1.0,
                 w0.ptr, w1.ptr, s);
      first = false;
    }
  }
  // single-time outputs: contract the owned time rows locally
  for (int I = 0; I < L.nb; I++) {
    if (by_out[I].empty() || L.ext(I)) continue;
    fill(Pall.ptr + poff[I], 0.0, L.spatial[I], s);
    for (int g : by_out[I]) {
      const Group& G = groups[g];
      const int rows = L.rows(G.tJ, me);
      if (rows == 0) continue;
      Gemm gm;  // partial[1 x S] += F0[0, row0 : row0 + rows] Z_q
      gm.M = 1; gm.N = (int)L.spatial[I]; gm.K = rows;
      gm.A = G.F0 + L.row0(G.tJ, me); gm.a_rs = G.n0J; gm.a_cs = 1;
      gm.B = Zall.ptr + G.zoff; gm.b_rs = L.spatial[I]; gm.b_cs = 1;
      gm.C = Pall.ptr + poff[I]; gm.c_rs = L.spatial[I]; gm.c_cs = 1;
      gm.beta = 1.0;
      run_gemm(gm, s);
    }
  }
  pack1.run(Zall.ptr, sendbuf, false, s);
}

void ShardOp::mid(const double* recvbuf, double* sendbuf, cudaStream_t s) {
  unpack1.run(recvbuf, Ball.ptr, false, s);
  const int me = L.rank;
  for (int I = 0; I < L.nb; I++) {
    if (by_out[I].empty() || !L.ext(I)) continue;
    const int64_t ch = L.chunk(I, me);
    if (ch == 0) continue;
    Gemm g;  // Y_I[n0 x chunk] = A_I[n0 x K] B_I[K x chunk]
    g.M = L.n0; g.N = (int)ch; g.K = (int)Kdim[I];
    g.A = A[I].ptr; g.a_rs = Kdim[I]; g.a_cs = 1;
    g.B = Ball.ptr + boff[I]; g.b_rs = ldc[I]; g.b_cs = 1;
    g.C = Yall.ptr + yoff[I]; g.c_rs = ldc[I]; g.c_cs = 1;
    run_gemm(g, s);
  }
  pack2y.run(Yall.ptr, sendbuf, false, s);
  pack2p.run(Pall.ptr, sendbuf, false, s);
}

// y = (noise x, by the caller) + received rows; rank 0 adds the single-time
// partials of every rank in rank order (deterministic)
void ShardOp::end(const double* recvbuf, double* y, cudaStream_t s) {
  unpack2.run(recvbuf, y, true, s);
  for (const auto& u : unpack2_single) u.run(recvbuf, y, true, s);
}

}  // namespace gpfvm

// ---- the sharded problem handle -------------------------------------------------
struct gpfvm_shard {
  gpfvm_problem* p = nullptr;
  gpfvm::ShardLayout L;
  int kind = 0;
  std::vector<std::unique_ptr<gpfvm::ShardOp>> ops;  // Gram: [G]; precond: [Q^T, Q]
  gpfvm::DevBuf noise_local, dinv_local;
  std::vector<gpfvm::BlockFD> keep_bj;  // precond: eigenbases referenced by single-time groups
};

namespace gpfvm {
namespace {

template <class F>
int guarded_shard(F&& f) {
  try {
    f();
    return GPFVM_OK;
  } catch (const Error& e) {
    set_error(e.msg);
    return e.code;
  } catch (const std::exception& e) {
    set_error(e.what());
    return GPFVM_ERR_INVALID;
  }
}

// time-site class of every block: blocks whose dimension-0 sites are equal
std::vector<int> time_classes(const gpfvm_problem* p) {
  std::vector<int> cls(p->blocks.size(), -1);
  int next = 0;
  for (size_t a = 0; a < p->blocks.size(); a++) {
    if (cls[a] >= 0) continue;
    cls[a] = next;
    const Sites& sa = p->blocks[a].sites[0];
    for (size_t b = a + 1; b < p->blocks.size(); b++) {
      const Sites& sb = p->blocks[b].sites[0];
      if (cls[b] < 0 && sa.kind == sb.kind && sa.lo == sb.lo && sa.hi == sb.hi) cls[b] = next;
    }
    next++;
  }
  return cls;
}

// local slab of a full block-concatenated vector (device), in the local layout
void gather_local(const ShardLayout& L, const gpfvm_problem* p, const double* full, double* local, cudaStream_t s) {
  for (int J = 0; J < L.nb; J++) {
    const int64_t rows = L.rows(J, L.rank);
    if (rows == 0) continue;
    GPFVM_CUDA(cudaMemcpyAsync(local + L.loc_off[J], full + p->blocks[J].offset + (int64_t)L.row0(J, L.rank) * L.spatial[J],
                               rows * L.spatial[J] * sizeof(double), cudaMemcpyDeviceToDevice, s));
  }
}

}  // namespace
}  // namespace gpfvm

namespace gpfvm {
// the Gram's Kronecker terms (R6 cancellation applied when the problem was
// created), keyed by the value of their time factor: (output, time classes, orders)
std::vector<ShardTermIn> gram_shard_terms(const gpfvm_problem* p) {
  const std::vector<int> tcls = time_classes(p);
  std::map<std::tuple<int, int, int, int, int>, int64_t> tk;
  std::map<int, std::tuple<int, int, int, int, int>> fid_key;
  for (const auto& kv : p->factor_index) {
    int out_, dim, bl, ml, br, mr;
    std::tie(out_, dim, bl, ml, br, mr) = kv.first;
    if (dim == 0) fid_key[kv.second] = std::make_tuple(out_, tcls[bl], ml, tcls[br], mr);
  }
  std::vector<ShardTermIn> terms;
  for (const auto& t : p->terms) {
    ShardTermIn st;
    st.I = t.I;
    st.J = t.J;
    st.coef = t.coef;
    for (int i = 0; i < p->ndim; i++) {
      st.f[i] = p->factors[t.fid[i]].data.ptr;
      st.sg[i] = p->factors[t.fid[i]].psign;
    }
    auto key = fid_key.at(t.fid[0]);
    auto it = tk.find(key);
    st.tkey = (it == tk.end()) ? (tk[key] = (int64_t)tk.size()) : it->second;
    terms.push_back(st);
  }
  return terms;
}
}  // namespace gpfvm

using namespace gpfvm;

extern "C" {

int gpfvm_shard_plan_counts(const gpfvm_problem* p, int rank, int world, int64_t* local_n, int64_t* send1,
                            int64_t* recv1, int64_t* send2, int64_t* recv2) {
  return guarded_shard([&] {
    GPFVM_CHECK(p && local_n, GPFVM_ERR_INVALID, "null argument");
    ShardOp op;
    op.plan(make_layout(p, rank, world), gram_shard_terms(p));
    *local_n = op.L.local_n;
    for (int r = 0; r < world; r++) {
      if (send1) send1[r] = op.send1[r];
      if (recv1) recv1[r] = op.recv1[r];
      if (send2) send2[r] = op.send2[r];
      if (recv2) recv2[r] = op.recv2[r];
    }
  });
}

int gpfvm_shard_create(gpfvm_problem* p, int rank, int world, int kind, gpfvm_shard** out, void* stream) {
  return guarded_shard([&] {
    GPFVM_CHECK(p && out, GPFVM_ERR_INVALID, "null argument");
    GPFVM_CHECK(p->assembled, GPFVM_ERR_STATE, "gpfvm_shard_create: call gpfvm_assemble_factors first");
    GPFVM_CHECK(kind == GPFVM_SHARD_GRAM || kind == GPFVM_SHARD_PRECOND, GPFVM_ERR_INVALID, "unknown shard kind");
    GPFVM_CUDA(cudaSetDevice(p->device));
    cudaStream_t s = (cudaStream_t)stream;
    auto sh = std::make_unique<gpfvm_shard>();
    sh->p = p;
    sh->kind = kind;
    sh->L = make_layout(p, rank, world);
    const ShardLayout& L = sh->L;
    const std::vector<int> tcls = time_classes(p);
    if (kind == GPFVM_SHARD_GRAM) {
      const std::vector<ShardTermIn> terms = gram_shard_terms(p);
      auto op = std::make_unique<ShardOp>();
      op->build(p, L, terms, {}, s);
      sh->ops.push_back(std::move(op));
      // local noise vector
      sh->noise_local.ensure((size_t)std::max<int64_t>(1, L.local_n));
      gather_local(L, p, p->noise.ptr, sh->noise_local.ptr, s);
    } else {
      // block-Jacobi fast diagonalisation: per block the
      // eigenbases Q_i (replicated: n_i x n_i eigensolves on every rank) and the
      // local slab of D^{-1}; P^{-1} = (x)Q  D^{-1}  (x)Q^T as two sharded
      // single-term operators around a local scaling
      std::vector<BlockFD> bj(p->blocks.size());
      PencilCache cache;
      for (int b = 0; b < (int)p->blocks.size(); b++) build_block_fd(p, b, bj[b], s, &cache);
      std::vector<ShardTermIn> fwd, bwd;
      for (int b = 0; b < (int)p->blocks.size(); b++) {
        ShardTermIn tf, tb;
        tf.I = tf.J = tb.I = tb.J = b;
        tf.coef = tb.coef = 1.0;
        tf.tkey = tb.tkey = b;
        for (int i = 0; i < p->ndim; i++) {
          tf.f[i] = bj[b].Qt[i].ptr;
          tb.f[i] = bj[b].Q[i].ptr;
        }
        fwd.push_back(tf);
        bwd.push_back(tb);
      }
      auto of = std::make_unique<ShardOp>(), ob = std::make_unique<ShardOp>();
      of->build(p, L, fwd, {}, s);
      ob->build(p, L, bwd, {}, s);
      // the ShardOps copied the time factors; the spatial KronSums keep
      // pointers to the Q's: move the BlockFD storage into the handle
      sh->dinv_local.ensure((size_t)std::max<int64_t>(1, L.local_n));
      for (int J = 0; J < L.nb; J++) {
        const int64_t rows = L.rows(J, rank);
        if (rows == 0) continue;
        GPFVM_CUDA(cudaMemcpyAsync(sh->dinv_local.ptr + L.loc_off[J], bj[J].Dinv.ptr + (int64_t)L.row0(J, rank) * L.spatial[J],
                                   rows * L.spatial[J] * sizeof(double), cudaMemcpyDeviceToDevice, s));
      }
      sh->ops.push_back(std::move(of));
      sh->ops.push_back(std::move(ob));
      GPFVM_CUDA(cudaStreamSynchronize(s));
      sh->keep_bj = std::move(bj);
    }
    *out = sh.release();
  });
}

int gpfvm_shard_destroy(gpfvm_shard* sh) {
  delete sh;
  return GPFVM_OK;
}

int64_t gpfvm_shard_local_size(const gpfvm_shard* sh) { return sh ? sh->L.local_n : -1; }

int gpfvm_shard_layout(const gpfvm_shard* sh, int64_t* local_offset, int64_t* row0, int64_t* rows, int64_t* spatial) {
  return guarded_shard([&] {
    GPFVM_CHECK(sh, GPFVM_ERR_INVALID, "null shard");
    for (int J = 0; J < sh->L.nb; J++) {
      if (local_offset) local_offset[J] = sh->L.loc_off[J];
      if (row0) row0[J] = sh->L.row0(J, sh->L.rank);
      if (rows) rows[J] = sh->L.rows(J, sh->L.rank);
      if (spatial) spatial[J] = sh->L.spatial[J];
    }
  });
}

int gpfvm_shard_counts(const gpfvm_shard* sh, int phase, int64_t* send1, int64_t* recv1, int64_t* send2, int64_t* recv2) {
  return guarded_shard([&] {
    GPFVM_CHECK(sh && phase >= 0 && phase < (int)sh->ops.size(), GPFVM_ERR_INVALID, "bad shard / phase");
    const ShardOp& op = *sh->ops[phase];
    for (int r = 0; r < sh->L.world; r++) {
      if (send1) send1[r] = op.send1[r];
      if (recv1) recv1[r] = op.recv1[r];
      if (send2) send2[r] = op.send2[r];
      if (recv2) recv2[r] = op.recv2[r];
    }
  });
}

int gpfvm_shard_apply_begin(gpfvm_shard* sh, int phase, const double* x_local, double* send1, void* stream) {
  return guarded_shard([&] {
    GPFVM_CHECK(sh && phase >= 0 && phase < (int)sh->ops.size() && x_local && send1, GPFVM_ERR_INVALID, "bad arguments");
    GPFVM_CUDA(cudaSetDevice(sh->p->device));
    sh->ops[phase]->begin(x_local, send1, (cudaStream_t)stream);
  });
}

int gpfvm_shard_apply_mid(gpfvm_shard* sh, int phase, const double* recv1, double* send2, void* stream) {
  return guarded_shard([&] {
    GPFVM_CHECK(sh && phase >= 0 && phase < (int)sh->ops.size() && recv1 && send2, GPFVM_ERR_INVALID, "bad arguments");
    GPFVM_CUDA(cudaSetDevice(sh->p->device));
    sh->ops[phase]->mid(recv1, send2, (cudaStream_t)stream);
  });
}

int gpfvm_shard_apply_end(gpfvm_shard* sh, int phase, const double* recv2, const double* x_local, double* y_local,
                          void* stream) {
  return guarded_shard([&] {
    GPFVM_CHECK(sh && phase >= 0 && phase < (int)sh->ops.size() && recv2 && y_local, GPFVM_ERR_INVALID, "bad arguments");
    GPFVM_CUDA(cudaSetDevice(sh->p->device));
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t n = sh->L.local_n;
    if (sh->kind == GPFVM_SHARD_GRAM) {
      GPFVM_CHECK(x_local, GPFVM_ERR_INVALID, "Gram end needs x_local (noise term)");
      if (n > 0) {
        shard_noise_kernel<<<gsz(n), 256, 0, s>>>(y_local, x_local, sh->noise_local.ptr, n);
        count_launch();
      }
    } else {
      fill(y_local, 0.0, n, s);
    }
    sh->ops[phase]->end(recv2, y_local, s);
    check_launch("gpfvm_shard_apply_end");
  });
}

int gpfvm_shard_precond_scale(gpfvm_shard* sh, double* z_local, void* stream) {
  return guarded_shard([&] {
    GPFVM_CHECK(sh && sh->kind == GPFVM_SHARD_PRECOND && z_local, GPFVM_ERR_INVALID, "bad arguments");
    const int64_t n = sh->L.local_n;
    if (n == 0) return;
    shard_vmul_kernel<<<gsz(n), 256, 0, (cudaStream_t)stream>>>(z_local, sh->dinv_local.ptr, n);
    count_launch();
    check_launch("gpfvm_shard_precond_scale");
  });
}

int gpfvm_shard_predict_mean(gpfvm_shard* sh, const gpfvm_grid* grid, const double* alpha_local, double* mean_partial,
                             void* stream) {
  return guarded_shard([&] {
    GPFVM_CHECK(sh && grid && alpha_local && mean_partial, GPFVM_ERR_INVALID, "null argument");
    gpfvm_problem* p = sh->p;
    GPFVM_CHECK(grid->output >= 0 && grid->output < p->nout, GPFVM_ERR_INVALID, "grid output out of range");
    for (int i = 0; i < p->ndim; i++)
      GPFVM_CHECK(grid->n[i] >= 1 && grid->pts[i], GPFVM_ERR_INVALID, "empty grid dimension");
    GPFVM_CUDA(cudaSetDevice(p->device));
    std::vector<int> row0(sh->L.nb), rows(sh->L.nb);
    for (int J = 0; J < sh->L.nb; J++) {
      row0[J] = sh->L.row0(J, sh->L.rank);
      rows[J] = sh->L.rows(J, sh->L.rank);
    }
    predict_mean_shard(p, *grid, alpha_local, sh->L.loc_off.data(), row0.data(), rows.data(), mean_partial,
                       (cudaStream_t)stream);
  });
}

int gpfvm_shard_gather_local(const gpfvm_shard* sh, const double* full, double* local, void* stream) {
  return guarded_shard([&] {
    GPFVM_CHECK(sh && full && local, GPFVM_ERR_INVALID, "bad arguments");
    gather_local(sh->L, sh->p, full, local, (cudaStream_t)stream);
  });
}

}  // extern "C"
