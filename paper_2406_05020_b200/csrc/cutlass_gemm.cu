// Plain batched FP64 GEMMs through CUTLASS's sm80 tensor-op DGEMM templates
// (DMMA.8x8x4 mainloop, 128x64x16 CTA tile, 64x32 warp tile, 4-stage cp.async
// pipeline) instantiated inside this library from the vendored CUTLASS
// headers.  Measured on this pool's B200 (scratch benchmark):
// 35 TF/s on the config-1 mode-product shapes vs 25-27 TF/s for the
// hand-written dgemm_dmma_kernel, which remains the path for K-segmented,
// multi-level-batched and tiny GEMMs.
#include "internal.h"

#ifdef GPFVM_WITH_CUTLASS
#include "cutlass/gemm/device/gemm_batched.h"

namespace gpfvm {

namespace {
template <class LayoutB>
using DGemm = cutlass::gemm::device::GemmBatched<
    double, cutlass::layout::RowMajor, double, LayoutB, double, cutlass::layout::RowMajor, double,
    cutlass::arch::OpClassTensorOp, cutlass::arch::Sm80, cutlass::gemm::GemmShape<128, 64, 16>,
    cutlass::gemm::GemmShape<64, 32, 16>, cutlass::gemm::GemmShape<8, 8, 4>,
    cutlass::epilogue::thread::LinearCombination<double, 1, double, double>,
    cutlass::gemm::threadblock::GemmBatchedIdentityThreadblockSwizzle, 4>;

template <class LayoutB>
bool launch(const Gemm& g, int64_t ldb, cudaStream_t s) {
  using Op = DGemm<LayoutB>;
  typename Op::Arguments args({g.M, g.N, g.K}, {g.A, g.a_rs}, (long long)g.a_b1, {g.B, ldb}, (long long)g.b_b1,
                              {g.C, g.c_rs}, (long long)g.c_b1, {g.C, g.c_rs}, (long long)g.c_b1, {g.alpha, g.beta},
                              g.batch1);
  Op op;
  if (op.can_implement(args) != cutlass::Status::kSuccess) return false;
  if (op(args, nullptr, s) != cutlass::Status::kSuccess) return false;
  count_launch();
  check_launch("cutlass dgemm");
  return true;
}
}  // namespace

bool try_cutlass_gemm(const Gemm& g, cudaStream_t s) {
  static const bool off = getenv("GPFVM_NO_CUTLASS") != nullptr;
  if (off) return false;
  if (g.nseg != 1 || g.batch2 != 1 || g.batch3 != 1) return false;
  if (g.a_cs != 1 || g.c_cs != 1) return false;
  if (g.M < 64 || g.N < 32 || g.K < 16) return false;
  // enough CTA tiles to fill the machine
  const int64_t tiles = ((g.M + 127) / 128) * (int64_t)((g.N + 63) / 64) * g.batch1;
  if (tiles < 148) return false;
  if (g.b_cs == 1) return launch<cutlass::layout::RowMajor>(g, g.b_rs, s);
  if (g.b_rs == 1) return launch<cutlass::layout::ColumnMajor>(g, g.b_cs, s);
  return false;
}

}  // namespace gpfvm

#else

namespace gpfvm {
bool try_cutlass_gemm(const Gemm&, cudaStream_t) { return false; }
}  // namespace gpfvm

#endif
