// dataset.cpp — grasps.jsonl and profile.json writers in the reference's
// result format (dataset.cpp:23-56, 113-131): nlohmann::json objects with
// keys in sorted order, compact dump, shortest round-trip doubles, the
// quaternion sign flip w < 0 -> -q.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <stdexcept>

#include "caller.hpp"

namespace lgh {

// Shortest round-trip decimal of v in nlohmann::json's number format
// (Grisu-style digits; fixed notation for exponents in (-4, 15], else
// d.ddde+XX with at least two exponent digits; integral values get ".0").
std::string json_double(double v) {
  if (!std::isfinite(v)) return "null";
  if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
  char buf[64];
  int prec = 1;
  for (; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof(buf), "%.*e", prec - 1, v);
    if (std::strtod(buf, nullptr) == v) break;
  }
  // buf = [-]d.ddde[+-]XX
  std::string s(buf);
  bool neg = s[0] == '-';
  if (neg) s = s.substr(1);
  size_t epos = s.find('e');
  int e10 = std::atoi(s.c_str() + epos + 1);
  std::string digits;
  for (size_t i = 0; i < epos; ++i)
    if (s[i] != '.') digits += s[i];
  while (digits.size() > 1 && digits.back() == '0') digits.pop_back();
  int k = (int)digits.size();
  int n = e10 + 1;  // position of the decimal point
  std::string out;
  if (k <= n && n <= 15) {
    out = digits + std::string(n - k, '0') + ".0";
  } else if (0 < n && n <= 15) {
    out = digits.substr(0, n) + "." + digits.substr(n);
  } else if (-4 < n && n <= 0) {
    out = "0." + std::string(-n, '0') + digits;
  } else {
    out = digits.substr(0, 1);
    if (k > 1) out += "." + digits.substr(1);
    int e = n - 1;
    out += "e";
    out += e < 0 ? "-" : "+";
    int ae = e < 0 ? -e : e;
    if (ae < 10) out += "0";
    out += std::to_string(ae);
  }
  return neg ? "-" + out : out;
}

namespace {

std::string vec(const double* v) {
  return "[" + json_double(v[0]) + "," + json_double(v[1]) + "," + json_double(v[2]) + "]";
}

// Eigen Quaternion from rotation matrix (Shepperd), w, x, y, z.
void quat_of(const double* R, double* q) {
  double m[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) m[i][j] = R[3 * i + j];
  double t = m[0][0] + m[1][1] + m[2][2];
  double c[4];  // x y z w (Eigen coeffs order)
  if (t > 0.0) {
    t = std::sqrt(t + 1.0);
    c[3] = 0.5 * t;
    t = 0.5 / t;
    c[0] = (m[2][1] - m[1][2]) * t;
    c[1] = (m[0][2] - m[2][0]) * t;
    c[2] = (m[1][0] - m[0][1]) * t;
  } else {
    int i = 0;
    if (m[1][1] > m[0][0]) i = 1;
    if (m[2][2] > m[i][i]) i = 2;
    int j = (i + 1) % 3;
    int k = (j + 1) % 3;
    t = std::sqrt(m[i][i] - m[j][j] - m[k][k] + 1.0);
    c[i] = 0.5 * t;
    t = 0.5 / t;
    c[3] = (m[k][j] - m[j][k]) * t;
    c[j] = (m[j][i] + m[i][j]) * t;
    c[k] = (m[k][i] + m[i][k]) * t;
  }
  if (c[3] < 0.0)
    for (double& x : c) x = -x;
  q[0] = c[3];
  q[1] = c[0];
  q[2] = c[1];
  q[3] = c[2];
}

}  // namespace

void write_dataset(const std::string& path, const lg_grasp* gs, long long n) {
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot write dataset: " + path);
  for (long long i = 0; i < n; ++i) {
    const lg_grasp& g = gs[i];
    double q[4];
    quat_of(g.pose_R, q);
    std::string s = "{\"contacts\":[";
    for (int c = 0; c < g.n_contacts; ++c) {
      if (c) s += ",";
      s += "{\"link\":" + std::to_string(g.contact_link[c]) + ",\"n\":" + vec(g.contact_n[c]) +
           ",\"p\":" + vec(g.contact_p[c]) + "}";
    }
    s += "],\"flags\":{\"ik_converged\":";
    s += g.ik_converged ? "true" : "false";
    s += ",\"penetration_free\":";
    s += g.penetration_free ? "true" : "false";
    s += ",\"stable\":";
    s += g.stable ? "true" : "false";
    s += "},\"objective\":" + json_double(g.objective) + ",\"pose\":[";
    s += json_double(q[0]) + "," + json_double(q[1]) + "," + json_double(q[2]) + "," +
         json_double(q[3]) + "," + json_double(g.pose_t[0]) + "," + json_double(g.pose_t[1]) +
         "," + json_double(g.pose_t[2]) + "],\"q\":[";
    for (int j = 0; j < g.dof; ++j) {
      if (j) s += ",";
      s += json_double(g.q[j]);
    }
    s += "]}";
    out << s << "\n";
  }
}

void write_profile(const std::string& path, const lg_profile& p) {  // dataset.cpp:113-131
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot write profile: " + path);
  out << "{\n"
      << "  \"candidates\": " << p.candidates << ",\n"
      << "  \"contact_optimization\": " << json_double(p.contact_optimization) << ",\n"
      << "  \"contact_sets_balanced\": " << p.contact_sets_balanced << ",\n"
      << "  \"grasps_per_second\": " << json_double(p.grasps_per_second) << ",\n"
      << "  \"ik_converged\": " << p.ik_converged << ",\n"
      << "  \"ik_finite\": " << p.ik_finite << ",\n"
      << "  \"kinematics_optimization\": " << json_double(p.kinematics_optimization) << ",\n"
      << "  \"penetration_free\": " << p.penetration_free << ",\n"
      << "  \"placement_domains\": " << json_double(p.placement_domains) << ",\n"
      << "  \"placements_accepted\": " << p.placements_accepted << ",\n"
      << "  \"postprocessing\": " << json_double(p.postprocessing) << ",\n"
      << "  \"stable\": " << p.stable << ",\n"
      << "  \"total\": " << json_double(p.total) << ",\n"
      << "  \"valid\": " << p.valid << "\n"
      << "}\n";
}

}  // namespace lgh
