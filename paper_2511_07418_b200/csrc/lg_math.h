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
//  2. The transcendentals of the hot path (sin, cos, log, atan2, hypot) as
//     glibc computes them (lg_libm.h): CUDA's libdevice and glibc differ in
//     the last ulp, and the contact search is chaotic (a one-ulp change in a
//     Box-Muller draw can flip a nearest-element argmin), so the device runs
//     glibc's own algorithms and reproduces the reference's host results bit
//     for bit (tests/test_libm.py: 0 mismatches).  sqrt, floor and division
//     are IEEE on both sides and need no substitute.
#pragma once

#include <stdint.h>
#include <math.h>

#include "lg_libm.h"

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

// ------------------------------------------------------------ transcendentals
// glibc 2.39's own algorithms (FMA builds), restated in lg_libm.h: the device
// and the oracle compute exactly what the reference's std::sin / std::cos /
// std::log / std::atan2 / std::hypot return on the host.
LG_HD double xsin(double x) { return lgl::xsin(x); }
LG_HD double xcos(double x) { return lgl::xcos(x); }
LG_HD double xlog(double x) { return lgl::xlog(x); }
LG_HD double xatan2(double y, double x) { return lgl::xatan2(y, x); }
LG_HD double xhypot(double x, double y) { return lgl::xhypot(x, y); }

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
