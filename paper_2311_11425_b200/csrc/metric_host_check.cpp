// Host build of the device metric arithmetic (metric_math.h), compiled with
// -ffp-contract=off.  Exported only for the CPU test suite, which checks it
// bit for bit against the reference's numpy metrics (tests/test_metric_order.py):
// the sm_100a kernel runs the same source with __dmul_rn/__dadd_rn, so a
// bitwise host match pins the kernel's operation order without a GPU.
// Never called by the product path.
#include <vector>

#include "hv_common.h"
#include "metric_math.h"

namespace {
struct NoBarrier {
  void operator()() const {}
};

template <int n>
void run(int scheme, const double* D, const double* coords, int64_t nelem, double* dx, double* J, double* grad) {
  constexpr int nn = n * n * n;
  std::vector<double> A(9 * nn), dxe(9 * nn);
  for (int64_t e = 0; e < nelem; ++e) {
    double* dxo = dx ? dx + e * 9 * nn : dxe.data();
    hv::element_metrics<n>(scheme, D, coords + e * 3 * nn, dxo, J + e * nn, A.data(), grad + e * 9 * nn, 0, 1,
                           NoBarrier{});
  }
}
}  // namespace

extern "C" int hv_debug_metric_terms_host(int scheme, int N, const double* h_D, const double* h_coords, int64_t nelem,
                                          double* h_dxdxi, double* h_J, double* h_grad) {
  if (!h_D || !h_coords || !h_J || !h_grad || nelem <= 0) HV_FAIL(HV_ERR_INVALID, "bad args");
  switch (N + 1) {
    case 2: run<2>(scheme, h_D, h_coords, nelem, h_dxdxi, h_J, h_grad); break;
    case 3: run<3>(scheme, h_D, h_coords, nelem, h_dxdxi, h_J, h_grad); break;
    case 4: run<4>(scheme, h_D, h_coords, nelem, h_dxdxi, h_J, h_grad); break;
    case 5: run<5>(scheme, h_D, h_coords, nelem, h_dxdxi, h_J, h_grad); break;
    case 6: run<6>(scheme, h_D, h_coords, nelem, h_dxdxi, h_J, h_grad); break;
    case 7: run<7>(scheme, h_D, h_coords, nelem, h_dxdxi, h_J, h_grad); break;
    case 8: run<8>(scheme, h_D, h_coords, nelem, h_dxdxi, h_J, h_grad); break;
    case 9: run<9>(scheme, h_D, h_coords, nelem, h_dxdxi, h_J, h_grad); break;
    default: HV_FAIL(HV_ERR_UNSUPPORTED, "degree %d", N);
  }
  return HV_OK;
}
