// Launch dispatch over the basis kinds (make_basis, basis.cpp:116-180) and
// the kernel shape query. The kernels and their constant tables live in
// sipg_gl.cu, sipg_gauss.cu and sipg_hermite.cu (sipg_launch.cuh).
#include "device.hpp"
#include "sipg_kernel.cuh"
#include "sipg_pairs.cuh"

namespace dgx
{

#define DGX_DECL(B)                                                                       \
  void upload_tables_##B(int K);                                                         \
  void launch_rhs_##B(int D, int K, bool compressed, bool adv,                           \
                      const dev::RhsParams<double> &prm, cudaStream_t s);                \
  void launch_adv_##B(int D, int K, bool compressed, const dev::AdvParams<double> &prm,   \
                      cudaStream_t s);                                                   \
  template <typename Real>                                                               \
  void launch_apply_##B(int D, int K, bool compressed, const dev::ApplyParams<Real> &prm, \
                        cudaStream_t s);
DGX_DECL(gl)
DGX_DECL(gauss)
DGX_DECL(hermite)
#undef DGX_DECL

void upload_tables(int K, int basis)
{
  switch (basis)
    {
    case 0: upload_tables_gl(K); break;
    case 1: upload_tables_gauss(K); break;
    case 2: upload_tables_hermite(K); break;
    default: fail(Code::invalid_argument, "unknown basis kind");
    }
}

int kernel_cells_per_cta(int D, int K, bool cart)
{
#define DGX_NC(DD, KK)                                                                     \
  if (D == DD && K == KK)                                                                  \
    return (DD == 3 && KK % 2 == 0) ? dev::PL<KK>::NC                                      \
           : cart                    ? dev::KernelShape<DD, KK, true, true>::NC            \
                                     : dev::KernelShape<DD, KK, true>::NC;
  DGX_NC(2, 2) DGX_NC(2, 3) DGX_NC(2, 4) DGX_NC(2, 5) DGX_NC(2, 6) DGX_NC(2, 7)
  DGX_NC(2, 8) DGX_NC(2, 9) DGX_NC(2, 10) DGX_NC(2, 11)
  DGX_NC(3, 2) DGX_NC(3, 3) DGX_NC(3, 4) DGX_NC(3, 5) DGX_NC(3, 6) DGX_NC(3, 7)
  DGX_NC(3, 8) DGX_NC(3, 9) DGX_NC(3, 10) DGX_NC(3, 11)
#undef DGX_NC
  return 1;
}

int kernel_brick(int D, int K)
{
#if defined(DGX_PAIRS) && !DGX_PAIRS
  (void)D, (void)K;
  return 0;
#else
#define DGX_BR(KK)                                                                         \
  if (D == 3 && K == KK)                                                                   \
    return dev::PL<KK>::BRICK;
  DGX_BR(2) DGX_BR(4) DGX_BR(6) DGX_BR(8) DGX_BR(10)
#undef DGX_BR
  return 0;
#endif
}

template <typename Real>
void launch_apply(int D, int K, int basis, bool compressed, const dev::ApplyParams<Real> &prm,
                  cudaStream_t s)
{
  switch (basis)
    {
    case 0: launch_apply_gl<Real>(D, K, compressed, prm, s); break;
    case 1: launch_apply_gauss<Real>(D, K, compressed, prm, s); break;
    case 2: launch_apply_hermite<Real>(D, K, compressed, prm, s); break;
    default: fail(Code::invalid_argument, "unknown basis kind");
    }
}

void launch_rhs(int D, int K, int basis, bool compressed, bool adv,
                const dev::RhsParams<double> &prm, cudaStream_t s)
{
  switch (basis)
    {
    case 0: launch_rhs_gl(D, K, compressed, adv, prm, s); break;
    case 1: launch_rhs_gauss(D, K, compressed, adv, prm, s); break;
    case 2: launch_rhs_hermite(D, K, compressed, adv, prm, s); break;
    default: fail(Code::invalid_argument, "unknown basis kind");
    }
}

void launch_adv(int D, int K, int basis, bool compressed, const dev::AdvParams<double> &prm,
                cudaStream_t s)
{
  switch (basis)
    {
    case 0: launch_adv_gl(D, K, compressed, prm, s); break;
    case 1: launch_adv_gauss(D, K, compressed, prm, s); break;
    case 2: launch_adv_hermite(D, K, compressed, prm, s); break;
    default: fail(Code::invalid_argument, "unknown basis kind");
    }
}

template void launch_apply<double>(int, int, int, bool, const dev::ApplyParams<double> &,
                                   cudaStream_t);
#ifdef DGX_WITH_FP32
template void launch_apply<float>(int, int, int, bool, const dev::ApplyParams<float> &,
                                  cudaStream_t);
#elif defined(DGX_DEV_K)
// kernel-experiment builds are fp64 only
template <>
void launch_apply<float>(int, int, int, bool, const dev::ApplyParams<float> &, cudaStream_t)
{
  fail(Code::invalid_argument, "fp32 apply not built (DGX_DEV_K experiment build)");
}
#endif

} // namespace dgx
