// Device Student-t CDF T_nu(y) for the score kernel (S2/S3 of SURVEY.md 8a).
//
// Same function and branch structure as the reference (dist.cpp:52-81):
//   x = nu / (y^2 + nu);  I = I_x(nu/2, 1/2);  T = y >= 0 ? 1 - I/2 : I/2
//   I_x(a,b) = front * CF(a,b,x)/a          for x <  (a+1)/(a+b+2)
//            = 1 - front * CF(b,a,1-x)/b    otherwise,
//   front = exp(a ln x + b ln(1-x) - ln B(a,b))
// but the continued fraction is evaluated division-free: the reference's modified Lentz
// spends ~6 FP64 divisions per iteration (dist.cpp:19-48); here the Wallis forward
// recurrence A_n = A_{n-1} + d_n A_{n-2} (same for B) runs on FMAs only, with the partial
// numerators d_n = coef_n * x read from host-computed coefficient tables.  The
// convergents B_n/A_n are the same continued-fraction convergents Lentz produces; the
// stopping rule |h_{2m+1}/h_{2m} - 1| < 1e-15 is tested through the determinant identity
// A_n B_{n-1} - A_{n-1} B_n = (-1)^n prod d_k, so no division is needed until the end.
#pragma once

#include "tie_internal.cuh"

namespace tie {
namespace dev {

// CF(p,q,x) = 1 / (1 + d1/(1 + d2/(1 + ...)))  (the value reference's incbeta_cf returns)
__device__ __forceinline__ double cf_wallis(const host::CfTable& t, double p, double q,
                                            double x) {
  // G = 1 + d1/(1 + d2/(...)):  A_{-1}=1, A_0=1, B_{-1}=0, B_0=1
  double d = t.d1 * x;
  double A_prev = 1.0, B_prev = 1.0;            // n = 0
  double A = 1.0 + d, B = 1.0;                  // n = 1
  // Fast path: tabulated coefficients, two iterations (four partial numerators) per
  // convergence test.  The test is the reference's |h_n / h_{n-1} - 1| < 1e-15 with
  // h = B/A, evaluated as |A_{n-1} B_n - A_n B_{n-1}| < 1e-15 |A_n B_{n-1}| (one FMA).
  // Iterating past the reference's stopping point only adds terms below 1e-15 relative.
  for (int m = 1; m + 1 <= host::CfTable::kTerms; m += 2) {
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      d = t.even[m - 1 + u] * x;
      double An = fma(d, A_prev, A), Bn = fma(d, B_prev, B);
      A_prev = A; B_prev = B; A = An; B = Bn;
      d = t.odd[m - 1 + u] * x;
      An = fma(d, A_prev, A); Bn = fma(d, B_prev, B);
      A_prev = A; B_prev = B; A = An; B = Bn;
    }
    const double c1 = A * B_prev;
    if (fabs(fma(A_prev, B, -c1)) < 1e-15 * fabs(c1)) return B / A;
  }
  // Slow path (extreme nu, x near the switch point): per-iteration test with the
  // determinant identity A_n B_{n-1} - A_{n-1} B_n = (-1)^n prod d_k, rescaling A, B.
  double det = fabs(fma(A, B_prev, -A_prev * B));
  for (int m = host::CfTable::kTerms + 1; m <= 100000; ++m) {
    const double m2 = 2.0 * m;
    const double ce = m * (q - m) / ((p - 1.0 + m2) * (p + m2));
    const double co = -(p + m) * (p + q + m) / ((p + m2) * (p + 1.0 + m2));
    // n = 2m (even numerator)
    d = ce * x;
    double An = fma(d, A_prev, A), Bn = fma(d, B_prev, B);
    A_prev = A; B_prev = B; A = An; B = Bn;
    det *= d;
    // n = 2m+1 (odd numerator)
    d = co * x;
    An = fma(d, A_prev, A); Bn = fma(d, B_prev, B);
    A_prev = A; B_prev = B; A = An; B = Bn;
    det *= d;
    // reference: del = h_{2m+1}/h_{2m};  |del - 1| = |det| / |A_{2m+1} B_{2m}|
    if (fabs(det) < 1e-15 * fabs(A * B_prev)) break;
    if ((m & 15) == 0) {  // keep A, B in range on very long fractions
      const double s = fabs(A);
      if (s > 1e150 || s < 1e-150) {
        const double r = 1.0 / s;
        A *= r; B *= r; A_prev *= r; B_prev *= r; det *= r * r;
      }
    }
  }
  return B / A;
}

__device__ __forceinline__ double t_cdf_dev(const TdistConst& td, double y) {
  if (isinf(y)) return y > 0.0 ? 1.0 : 0.0;
  // operation order mirrors dist.cpp:77 / dist.cpp:58 (no FMA contraction)
  const double x = td.nu / __dadd_rn(__dmul_rn(y, y), td.nu);
  double I;
  if (x == 0.0) {
    I = 0.0;
  } else if (x == 1.0) {
    I = 1.0;
  } else {
    const double front = exp(__dsub_rn(
        __dadd_rn(__dmul_rn(td.a, log(x)), __dmul_rn(td.b, log1p(-x))), td.logbeta));
    if (x < td.thresh)
      I = __dmul_rn(front, cf_wallis(td.ab, td.a, td.b, x)) / td.a;
    else
      I = __dsub_rn(1.0, __dmul_rn(front, cf_wallis(td.ba, td.b, td.a, 1.0 - x)) / td.b);
  }
  return y >= 0.0 ? __dsub_rn(1.0, 0.5 * I) : 0.5 * I;
}

}  // namespace dev
}  // namespace tie
