// lg_math.h — FP64 primitives shared by the CUDA kernels and the CPU oracle.
//
// Two things live here and nothing else:
//
//  1. The Eigen operations the reference uses (Vector3d / Matrix3d arithmetic,
//     AngleAxisd::toRotationMatrix, Quaterniond::toRotationMatrix), written out
//     in one canonical left-to-right evaluation order with no fused
//     multiply-add.  The reference's arithmetic is carried by Eigen
//     (SURVEY.md 8(c) "Third-party arithmetic"); bit-level parity with a
//     particular Eigen build is unpinned, so both of our restatements pin to
//     this order instead.  Device code is compiled with --fmad=false and the
//     oracle with -ffp-contract=off so that `a*b + c` is two IEEE roundings on
//     both sides.
//
//  2. A deterministic libm (sin, cos, log, atan2, hypot) used on the hot path
//     by both sides.  glibc and CUDA's libdevice differ in the last ulp, and the
//     contact search is chaotic (a one-ulp change in a Box-Muller draw can flip
//     a nearest-element argmin), so the device and the oracle must evaluate the
//     same function.  These follow the classic fdlibm argument reductions and
//     minimax kernels; tests/test_oracle_pins.py bounds their error against
//     glibc (<= 1 ulp) so the oracle stays a faithful stand-in for the
//     reference's glibc calls.  sqrt, floor and division are IEEE on both
//     sides and need no substitute.
#pragma once

#include <stdint.h>
#include <math.h>

#if defined(__CUDACC__)
#define LG_HD __host__ __device__ __forceinline__
#else
#define LG_HD static inline
#endif

namespace lgm {

// ---------------------------------------------------------------- bit access
LG_HD int64_t bits_of(double x) {
#if defined(__CUDA_ARCH__)
  return __double_as_longlong(x);
#else
  int64_t i;
  __builtin_memcpy(&i, &x, 8);
  return i;
#endif
}
LG_HD double from_bits(int64_t i) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double(i);
#else
  double x;
  __builtin_memcpy(&x, &i, 8);
  return x;
#endif
}
LG_HD int32_t high_word(double x) { return (int32_t)(bits_of(x) >> 32); }
LG_HD uint32_t low_word(double x) { return (uint32_t)(bits_of(x) & 0xffffffffu); }
LG_HD double with_high_word(double x, int32_t hi) {
  return from_bits(((int64_t)(uint32_t)hi << 32) | (int64_t)low_word(x));
}
LG_HD bool is_finite(double x) {
  return (bits_of(x) & 0x7ff0000000000000ll) != 0x7ff0000000000000ll;
}
LG_HD bool is_nan(double x) { return x != x; }
LG_HD double dabs(double x) { return from_bits(bits_of(x) & 0x7fffffffffffffffll); }

// std::max / std::min / std::clamp semantics (first argument on ties/NaN).
LG_HD double dmax(double a, double b) { return (a < b) ? b : a; }
LG_HD double dmin(double a, double b) { return (b < a) ? b : a; }
LG_HD double dclamp(double v, double lo, double hi) {
  return (v < lo) ? lo : (hi < v) ? hi : v;
}

// ------------------------------------------------------------------ sin/cos
// Argument reduction by Cody-Waite with pi/2 split into 33-bit pieces (fdlibm
// constants), result as a double-double (y0, y1); exact enough for |x| below
// ~2^20 * pi/2, far beyond anything the pipeline produces (joint angles, roll
// and Box-Muller phases are all within [-2pi, 2pi]).
LG_HD int rem_pio2(double x, double* y0, double* y1) {
  const double invpio2 = 6.36619772367581382433e-01;
  const double pio2_1 = 1.57079632673412561417e+00;
  const double pio2_1t = 6.07710050650619224932e-11;
  const double pio2_2 = 6.07710050630396597660e-11;
  const double pio2_2t = 2.02226624879595063154e-21;
  const double pio2_3 = 2.02226624871116645580e-21;
  const double pio2_3t = 8.47842766036889956997e-32;
  (void)pio2_1t;
  double ax = dabs(x);
  if (ax <= 7.85398163397448278999e-01) {  // |x| <= pi/4
    *y0 = x;
    *y1 = 0.0;
    return 0;
  }
  double t = x * invpio2;
  // round half away from zero, like (int)(t + copysign(0.5, t))
  double fn = (t >= 0.0) ? floor(t + 0.5) : -floor(-t + 0.5);
  int n = (int)fn;
  double r = x - fn * pio2_1;
  double w = fn * pio2_2;
  double tt = r;
  r = tt - w;
  w = fn * pio2_2t - ((tt - r) - w);
  double y = r - w;
  // third round for large fn where cancellation ate the second round
  int ex = (int)((high_word(x) >> 20) & 0x7ff);
  int ey = (int)((high_word(y) >> 20) & 0x7ff);
  if (ex - ey > 49) {
    tt = r;
    w = fn * pio2_3;
    r = tt - w;
    w = fn * pio2_3t - ((tt - r) - w);
    y = r - w;
  }
  *y0 = y;
  *y1 = (r - y) - w;
  return n;
}

LG_HD double k_sin(double x, double y, int iy) {
  const double S1 = -1.66666666666666324348e-01;
  const double S2 = 8.33333333332248946124e-03;
  const double S3 = -1.98412698298579493134e-04;
  const double S4 = 2.75573137070700676789e-06;
  const double S5 = -2.50507602534068634195e-08;
  const double S6 = 1.58969099521155010221e-10;
  double z = x * x;
  double w = z * z;
  double r = S2 + z * (S3 + z * S4) + z * w * (S5 + z * S6);
  double v = z * x;
  if (iy == 0) return x + v * (S1 + z * r);
  return x - ((z * (0.5 * y - v * r) - y) - v * S1);
}

LG_HD double k_cos(double x, double y) {
  const double C1 = 4.16666666666666019037e-02;
  const double C2 = -1.38888888888741095749e-03;
  const double C3 = 2.48015872894767294178e-05;
  const double C4 = -2.75573143513906633035e-07;
  const double C5 = 2.08757232129817482790e-09;
  const double C6 = -1.13596475577881948265e-11;
  double z = x * x;
  double w = z * z;
  double r = z * (C1 + z * (C2 + z * C3)) + w * w * (C4 + z * (C5 + z * C6));
  double hz = 0.5 * z;
  w = 1.0 - hz;
  return w + (((1.0 - w) - hz) + (z * r - x * y));
}

LG_HD double xsin(double x) {
#if defined(LG_USE_GLIBC) && !defined(__CUDA_ARCH__)
  return ::sin(x);
#endif
  if (!is_finite(x)) return x - x;
  if (dabs(x) < 7.450580596923828125e-09) return x;  // 2^-27
  double y0, y1;
  int n = rem_pio2(x, &y0, &y1);
  switch (n & 3) {
    case 0: return k_sin(y0, y1, 1);
    case 1: return k_cos(y0, y1);
    case 2: return -k_sin(y0, y1, 1);
    default: return -k_cos(y0, y1);
  }
}

LG_HD double xcos(double x) {
#if defined(LG_USE_GLIBC) && !defined(__CUDA_ARCH__)
  return ::cos(x);
#endif
  if (!is_finite(x)) return x - x;
  if (dabs(x) < 7.450580596923828125e-09) return 1.0;
  double y0, y1;
  int n = rem_pio2(x, &y0, &y1);
  switch (n & 3) {
    case 0: return k_cos(y0, y1);
    case 1: return -k_sin(y0, y1, 1);
    case 2: return -k_cos(y0, y1);
    default: return k_sin(y0, y1, 1);
  }
}

// ---------------------------------------------------------------------- log
LG_HD double xlog(double x) {
#if defined(LG_USE_GLIBC) && !defined(__CUDA_ARCH__)
  return ::log(x);
#endif
  const double ln2_hi = 6.93147180369123816490e-01;
  const double ln2_lo = 1.90821492927058770002e-10;
  const double two54 = 1.80143985094819840000e+16;
  const double Lg1 = 6.666666666666735130e-01;
  const double Lg2 = 3.999999999940941908e-01;
  const double Lg3 = 2.857142874366239149e-01;
  const double Lg4 = 2.222219843214978396e-01;
  const double Lg5 = 1.818357216161805012e-01;
  const double Lg6 = 1.531383769920937332e-01;
  const double Lg7 = 1.479819860511658591e-01;
  int32_t hx = high_word(x);
  uint32_t lx = low_word(x);
  int k = 0;
  if (hx < 0x00100000) {  // x < 2^-1022
    if (((hx & 0x7fffffff) | (int32_t)lx) == 0) return -__builtin_huge_val();  // -inf
    if (hx < 0) return (x - x) / (x - x);                              // NaN
    k -= 54;
    x *= two54;
    hx = high_word(x);
  }
  if (hx >= 0x7ff00000) return x + x;
  k += (hx >> 20) - 1023;
  hx &= 0x000fffff;
  int32_t i = (hx + 0x95f64) & 0x100000;
  x = with_high_word(x, hx | (i ^ 0x3ff00000));  // normalize x or x/2
  k += (i >> 20);
  double f = x - 1.0;
  double dk;
  if ((0x000fffff & (2 + hx)) < 3) {  // -2^-20 <= f < 2^-20
    if (f == 0.0) {
      if (k == 0) return 0.0;
      dk = (double)k;
      return dk * ln2_hi + dk * ln2_lo;
    }
    double R = f * f * (0.5 - 0.33333333333333333 * f);
    if (k == 0) return f - R;
    dk = (double)k;
    return dk * ln2_hi - ((R - dk * ln2_lo) - f);
  }
  double s = f / (2.0 + f);
  dk = (double)k;
  double z = s * s;
  i = hx - 0x6147a;
  double w = z * z;
  int32_t j = 0x6b851 - hx;
  double t1 = w * (Lg2 + w * (Lg4 + w * Lg6));
  double t2 = z * (Lg1 + w * (Lg3 + w * (Lg5 + w * Lg7)));
  i |= j;
  double R = t2 + t1;
  if (i > 0) {
    double hfsq = 0.5 * f * f;
    if (k == 0) return f - (hfsq - s * (hfsq + R));
    return dk * ln2_hi - ((hfsq - (s * (hfsq + R) + dk * ln2_lo)) - f);
  }
  if (k == 0) return f - s * (f - R);
  return dk * ln2_hi - ((s * (f - R) - dk * ln2_lo) - f);
}

// -------------------------------------------------------------- atan, atan2
LG_HD double xatan(double x) {
  const double atanhi[4] = {4.63647609000806093515e-01, 7.85398163397448278999e-01,
                            9.82793723247329054082e-01, 1.57079632679489655800e+00};
  const double atanlo[4] = {2.26987774529616870924e-17, 3.06161699786838301793e-17,
                            1.39033110312309984516e-17, 6.12323399573676603587e-17};
  const double aT[11] = {3.33333333333329318027e-01, -1.99999999998764832476e-01,
                         1.42857142725034663711e-01, -1.11111104054623557880e-01,
                         9.09088713343650656196e-02, -7.69187620504482999495e-02,
                         6.66107313738753120669e-02, -5.83357013379057348645e-02,
                         4.97687799461593236017e-02, -3.65315727442169155270e-02,
                         1.62858201153657823623e-02};
  int32_t hx = high_word(x);
  int32_t ix = hx & 0x7fffffff;
  int id;
  if (ix >= 0x44100000) {  // |x| >= 2^66
    if (is_nan(x)) return x + x;
    return (hx > 0) ? atanhi[3] + atanlo[3] : -atanhi[3] - atanlo[3];
  }
  if (ix < 0x3fdc0000) {  // |x| < 0.4375
    if (ix < 0x3e400000) return x;  // |x| < 2^-27
    id = -1;
  } else {
    x = dabs(x);
    if (ix < 0x3ff30000) {    // |x| < 1.1875
      if (ix < 0x3fe60000) {  // 7/16 <= |x| < 11/16
        id = 0;
        x = (2.0 * x - 1.0) / (2.0 + x);
      } else {  // 11/16 <= |x| < 19/16
        id = 1;
        x = (x - 1.0) / (x + 1.0);
      }
    } else {
      if (ix < 0x40038000) {  // |x| < 2.4375
        id = 2;
        x = (x - 1.5) / (1.0 + 1.5 * x);
      } else {  // 2.4375 <= |x| < 2^66
        id = 3;
        x = -1.0 / x;
      }
    }
  }
  double z = x * x;
  double w = z * z;
  double s1 = z * (aT[0] + w * (aT[2] + w * (aT[4] + w * (aT[6] + w * (aT[8] + w * aT[10])))));
  double s2 = w * (aT[1] + w * (aT[3] + w * (aT[5] + w * (aT[7] + w * aT[9]))));
  if (id < 0) return x - x * (s1 + s2);
  z = atanhi[id] - ((x * (s1 + s2) - atanlo[id]) - x);
  return (hx < 0) ? -z : z;
}

LG_HD double xatan2(double y, double x) {
#if defined(LG_USE_GLIBC) && !defined(__CUDA_ARCH__)
  return ::atan2(y, x);
#endif
  const double pi_o_4 = 7.8539816339744827900e-01;
  const double pi_o_2 = 1.5707963267948965580e+00;
  const double pi = 3.1415926535897931160e+00;
  const double pi_lo = 1.2246467991473531772e-16;
  if (is_nan(x) || is_nan(y)) return x + y;
  if (x == 1.0) return xatan(y);
  int32_t hx = high_word(x), hy = high_word(y);
  int32_t ix = hx & 0x7fffffff, iy = hy & 0x7fffffff;
  int m = ((hy >> 31) & 1) | ((hx >> 30) & 2);
  if (y == 0.0) {
    switch (m) {
      case 0:
      case 1: return y;
      case 2: return pi;
      default: return -pi;
    }
  }
  if (x == 0.0) return (hy < 0) ? -pi_o_2 : pi_o_2;
  if (!is_finite(x)) {
    if (!is_finite(y)) {
      switch (m) {
        case 0: return pi_o_4;
        case 1: return -pi_o_4;
        case 2: return 3.0 * pi_o_4;
        default: return -3.0 * pi_o_4;
      }
    }
    switch (m) {
      case 0: return 0.0;
      case 1: return -0.0;
      case 2: return pi;
      default: return -pi;
    }
  }
  if (!is_finite(y)) return (hy < 0) ? -pi_o_2 : pi_o_2;
  int k = (iy - ix) >> 20;
  double z;
  if (k > 60) {
    z = pi_o_2 + 0.5 * pi_lo;
    m &= 1;
  } else if (hx < 0 && k < -60) {
    z = 0.0;
  } else {
    z = xatan(dabs(y / x));
  }
  switch (m) {
    case 0: return z;
    case 1: return -z;
    case 2: return pi - (z - pi_lo);
    default: return (z - pi_lo) - pi;
  }
}

// -------------------------------------------------------------------- hypot
LG_HD double xhypot(double x, double y) {
#if defined(LG_USE_GLIBC) && !defined(__CUDA_ARCH__)
  return ::hypot(x, y);
#endif
  double a = dabs(x), b = dabs(y);
  if (!is_finite(a) || !is_finite(b)) {
    if (a == 1.0 / 0.0 || b == 1.0 / 0.0) return 1.0 / 0.0;
    return a + b;
  }
  if (a < b) {
    double t = a;
    a = b;
    b = t;
  }
  if (b == 0.0) return a;
  // exact power-of-two rescaling keeps a*a and b*b in range
  if (a > 1e150) {
    a *= 0x1p-600;
    b *= 0x1p-600;
    return sqrt(a * a + b * b) * 0x1p600;
  }
  if (b < 1e-150) {
    a *= 0x1p600;
    b *= 0x1p600;
    return sqrt(a * a + b * b) * 0x1p-600;
  }
  return sqrt(a * a + b * b);
}

// ----------------------------------------------------------- Eigen-like 3D
struct V3 {
  double x, y, z;
};
struct M3 {
  double m[9];  // row-major
};

LG_HD V3 v3(double x, double y, double z) {
  V3 r;
  r.x = x;
  r.y = y;
  r.z = z;
  return r;
}
LG_HD V3 v3_load(const double* p) { return v3(p[0], p[1], p[2]); }
LG_HD void v3_store(double* p, V3 a) {
  p[0] = a.x;
  p[1] = a.y;
  p[2] = a.z;
}
LG_HD double comp(V3 a, int i) { return i == 0 ? a.x : (i == 1 ? a.y : a.z); }
LG_HD V3 add(V3 a, V3 b) { return v3(a.x + b.x, a.y + b.y, a.z + b.z); }
LG_HD V3 sub(V3 a, V3 b) { return v3(a.x - b.x, a.y - b.y, a.z - b.z); }
LG_HD V3 neg(V3 a) { return v3(-a.x, -a.y, -a.z); }
LG_HD V3 scale(double s, V3 a) { return v3(s * a.x, s * a.y, s * a.z); }
LG_HD V3 divs(V3 a, double s) { return v3(a.x / s, a.y / s, a.z / s); }
LG_HD V3 cmul(V3 a, V3 b) { return v3(a.x * b.x, a.y * b.y, a.z * b.z); }
// a + s*b, per component (Eigen `a + s * b`)
LG_HD V3 axpy(V3 a, double s, V3 b) { return v3(a.x + s * b.x, a.y + s * b.y, a.z + s * b.z); }
LG_HD double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
LG_HD double sqnorm(V3 a) { return a.x * a.x + a.y * a.y + a.z * a.z; }
LG_HD double norm(V3 a) { return sqrt(sqnorm(a)); }
LG_HD V3 cross(V3 a, V3 b) {
  return v3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
// Eigen normalized(): divide by sqrt(squaredNorm) when > 0.
LG_HD V3 normalized(V3 a) {
  double z = sqnorm(a);
  if (z > 0.0) return divs(a, sqrt(z));
  return a;
}
LG_HD V3 vmin(V3 a, V3 b) { return v3(dmin(a.x, b.x), dmin(a.y, b.y), dmin(a.z, b.z)); }
LG_HD V3 vmax(V3 a, V3 b) { return v3(dmax(a.x, b.x), dmax(a.y, b.y), dmax(a.z, b.z)); }

LG_HD M3 m3_identity() {
  M3 r;
  for (int i = 0; i < 9; ++i) r.m[i] = (i % 4 == 0) ? 1.0 : 0.0;
  return r;
}
LG_HD M3 m3_load(const double* p) {
  M3 r;
  for (int i = 0; i < 9; ++i) r.m[i] = p[i];
  return r;
}
LG_HD void m3_store(double* p, const M3& a) {
  for (int i = 0; i < 9; ++i) p[i] = a.m[i];
}
LG_HD V3 mul(const M3& a, V3 v) {
  return v3(a.m[0] * v.x + a.m[1] * v.y + a.m[2] * v.z,
            a.m[3] * v.x + a.m[4] * v.y + a.m[5] * v.z,
            a.m[6] * v.x + a.m[7] * v.y + a.m[8] * v.z);
}
LG_HD M3 mul(const M3& a, const M3& b) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      r.m[3 * i + j] = a.m[3 * i] * b.m[j] + a.m[3 * i + 1] * b.m[3 + j] +
                       a.m[3 * i + 2] * b.m[6 + j];
  return r;
}
LG_HD M3 transpose(const M3& a) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r.m[3 * i + j] = a.m[3 * j + i];
  return r;
}

// Eigen's 3x3 determinant (cofactor expansion down the first column).
LG_HD double det3(const M3& a) {
  const double* m = a.m;
  double t0 = m[0] * (m[4] * m[8] - m[5] * m[7]);
  double t1 = m[3] * (m[1] * m[8] - m[2] * m[7]);
  double t2 = m[6] * (m[1] * m[5] - m[2] * m[4]);
  return (t0 - t1) + t2;
}

// RigidTransform::orthonormal_error (geometry.hpp:53-59):
// max(max |R R^T - I|, |det R - 1|).
LG_HD double orthonormal_error(const M3& r) {
  M3 p = mul(r, transpose(r));
  double e = 0.0;
  for (int i = 0; i < 9; ++i) {
    double v = dabs(p.m[i] - ((i % 4 == 0) ? 1.0 : 0.0));
    e = (i == 0 || v > e) ? v : e;
  }
  double d = dabs(det3(r) - 1.0);
  return dmax(e, d);
}

// Eigen AngleAxis<double>::toRotationMatrix (axis used as given).
LG_HD M3 angle_axis(double angle, V3 axis) {
  double s = lgm::xsin(angle);
  double c = lgm::xcos(angle);
  V3 sin_axis = scale(s, axis);
  V3 cos1_axis = scale(1.0 - c, axis);
  M3 r;
  double tmp;
  tmp = cos1_axis.x * axis.y;
  r.m[1] = tmp - sin_axis.z;
  r.m[3] = tmp + sin_axis.z;
  tmp = cos1_axis.x * axis.z;
  r.m[2] = tmp + sin_axis.y;
  r.m[6] = tmp - sin_axis.y;
  tmp = cos1_axis.y * axis.z;
  r.m[5] = tmp - sin_axis.x;
  r.m[7] = tmp + sin_axis.x;
  r.m[0] = cos1_axis.x * axis.x + c;
  r.m[4] = cos1_axis.y * axis.y + c;
  r.m[8] = cos1_axis.z * axis.z + c;
  return r;
}

// Eigen Quaternion<double>::toRotationMatrix (w, x, y, z), unnormalized input.
LG_HD M3 quat_to_matrix(double w, double x, double y, double z) {
  double tx = 2.0 * x, ty = 2.0 * y, tz = 2.0 * z;
  double twx = tx * w, twy = ty * w, twz = tz * w;
  double txx = tx * x, txy = ty * x, txz = tz * x;
  double tyy = ty * y, tyz = tz * y, tzz = tz * z;
  M3 r;
  r.m[0] = 1.0 - (tyy + tzz);
  r.m[1] = txy - twz;
  r.m[2] = txz + twy;
  r.m[3] = txy + twz;
  r.m[4] = 1.0 - (txx + tzz);
  r.m[5] = tyz - twx;
  r.m[6] = txz - twy;
  r.m[7] = tyz + twx;
  r.m[8] = 1.0 - (txx + tyy);
  return r;
}

// RigidTransform (geometry.hpp:28-62).
struct Xf {
  M3 R;
  V3 t;
};
LG_HD Xf xf_identity() {
  Xf x;
  x.R = m3_identity();
  x.t = v3(0.0, 0.0, 0.0);
  return x;
}
LG_HD V3 xf_apply(const Xf& a, V3 p) { return add(mul(a.R, p), a.t); }
LG_HD V3 xf_rotate(const Xf& a, V3 v) { return mul(a.R, v); }
LG_HD Xf xf_compose(const Xf& a, const Xf& b) {
  Xf r;
  r.R = mul(a.R, b.R);
  r.t = add(mul(a.R, b.t), a.t);
  return r;
}
LG_HD Xf xf_inverse(const Xf& a) {
  Xf r;
  r.R = transpose(a.R);
  r.t = neg(mul(r.R, a.t));
  return r;
}

// ------------------------------------------------------------ mt19937_64
// std::mt19937_64 ([rand.eng.mers] with the [rand.predef] parameters) with
// the state twisted lazily, one word per draw, in place.  The standard's
// block twist walks i = 0..311 updating mt[i] from mt[i], mt[i+1] and
// mt[(i+156)%312]; doing the same update for word i just before word i is
// emitted reads exactly the same (old or already-updated) neighbours, so the
// output sequence is identical while the per-draw cost stays flat.
struct Mt64 {
  uint64_t mt[312];
  int idx;
};
LG_HD void mt_seed(Mt64& g, uint64_t seed) {
  g.mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g.mt[i] = 6364136223846793005ull * (g.mt[i - 1] ^ (g.mt[i - 1] >> 62)) + (uint64_t)i;
  g.idx = 0;
}
LG_HD uint64_t mt_next(Mt64& g) {
  const uint64_t UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull;
  int i = g.idx;
  uint64_t y = (g.mt[i] & UM) | (g.mt[(i + 1 == 312) ? 0 : i + 1] & LM);
  int j = i + 156;
  if (j >= 312) j -= 312;
  uint64_t w = g.mt[j] ^ (y >> 1) ^ ((y & 1ull) ? 0xB5026F5AA96619E9ull : 0ull);
  g.mt[i] = w;
  g.idx = (i + 1 == 312) ? 0 : i + 1;
  uint64_t z = w;
  z ^= (z >> 29) & 0x5555555555555555ull;
  z ^= (z << 17) & 0x71D67FFFEDA60000ull;
  z ^= (z << 37) & 0xFFF7EEE000000000ull;
  z ^= (z >> 43);
  return z;
}

// splitmix mix64 / mix_seed (rng.hpp:16-28).
LG_HD uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d9b9b3f794a2e5ull;
  return x ^ (x >> 31);
}
LG_HD uint64_t mix_seed(uint64_t seed, uint64_t a, uint64_t b) {
  return mix64(mix64(seed ^ mix64(a)) ^ mix64(b ^ 0x5851f42d4c957f2dull));
}

// Rng distributions (rng.hpp:39-89) on top of a raw u64 draw.
LG_HD double u01(uint64_t u) { return (double)(u >> 11) * 0x1.0p-53; }

}  // namespace lgm
