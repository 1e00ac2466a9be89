// capi_core.cpp — host half of the product C-ABI (include/lg.h): the
// thread-local error message, the seed mixer and the validate_dataset issue
// texts.  Everything else lives in the device translation unit.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>

#include "capi_common.hpp"
#include "lg_math.h"

namespace lgc {
thread_local std::string g_error;
void set_error(const std::string& msg) { g_error = msg; }
}  // namespace lgc

using lgc::guard;

extern "C" {

int lg_last_error(char* buf, size_t cap) {
  if (buf && cap) {
    std::strncpy(buf, lgc::g_error.c_str(), cap - 1);
    buf[cap - 1] = 0;
  }
  return (int)lgc::g_error.size();
}

uint64_t lg_mix_seed(uint64_t seed, uint64_t a, uint64_t b) { return lgm::mix_seed(seed, a, b); }

// index_cache_key (config.cpp:403-417): FNV-1a (contact_field.cpp:486-494)
// over the hand file's bytes, then the index-shaping parameters.  The GGCF
// cache (lg_field_save / lg_field_load, run_batch with cache = 1) is keyed by it.
int lg_index_cache_key(const lg_run_params* c, uint64_t* key) {
  return guard([&] {
    if (!c || !key) throw std::invalid_argument("lg_index_cache_key: null argument");
    auto fnv1a = [](const void* data, size_t n, uint64_t h) {
      const unsigned char* b = (const unsigned char*)data;
      for (size_t i = 0; i < n; ++i) {
        h ^= b[i];
        h *= 0x100000001b3ull;
      }
      return h;
    };
    std::ifstream in(c->hand, std::ios::binary);
    if (!in) throw std::runtime_error(std::string("hash_file: cannot open ") + c->hand);
    uint64_t h = 0xcbf29ce484222325ull;
    char buf[4096];
    while (in.read(buf, sizeof(buf)) || in.gcount() > 0) h = fnv1a(buf, (size_t)in.gcount(), h);
    h = fnv1a(&c->seed, sizeof(c->seed), h);
    h = fnv1a(&c->field_configs, sizeof(c->field_configs), h);
    h = fnv1a(&c->box_width, sizeof(c->box_width), h);
    h = fnv1a(&c->patch_radius, sizeof(c->patch_radius), h);
    h = fnv1a(&c->field_points_per_patch, sizeof(c->field_points_per_patch), h);
    h = fnv1a(&c->codebook_size, sizeof(c->codebook_size), h);
    h = fnv1a(&c->samples_per_cm2, sizeof(c->samples_per_cm2), h);
    h = fnv1a(&c->hand_scale, sizeof(c->hand_scale), h);
    *key = h;
  });
}

// ValidationReport issue texts (validate.cpp:56-175); numbers as an ostream
// with default formatting prints them (%g, 6 significant digits).
int lg_validation_issues(const char* const* joint_names, int n_links,
                         const lg_grasp_check* checks, long long n, const lg_run_params* p,
                         char* buf, size_t cap, size_t* needed, long long* n_issues) {
  return guard([&] {
    if ((!joint_names && n_links) || (!checks && n) || !p)
      throw std::invalid_argument("lg_validation_issues: null argument");
    std::string out;
    long long count = 0;
    auto num = [](double v) {
      char t[64];
      std::snprintf(t, sizeof(t), "%g", v);
      return std::string(t);
    };
    auto add = [&](long long gi, const std::string& what) {
      out += std::to_string(gi) + "\t" + what + "\n";
      ++count;
    };
    for (long long gi = 0; gi < n; ++gi) {
      const lg_grasp_check& c = checks[gi];
      if (c.status == 1) {
        add(gi, "joint vector size mismatch");
        continue;
      }
      if (c.status == 2) {
        add(gi, "pose not rigid: transform rotation is not orthonormal");
        continue;
      }
      if (c.status == 3) {
        for (int k = 0; k < c.n_limit; ++k) {
          int l = c.limit_link[k];
          std::string name = (l >= 0 && l < n_links && joint_names[l]) ? joint_names[l] : std::string("?");
          add(gi, "joint " + name + " out of limits: " + num(c.limit_value[k]));
        }
        continue;
      }
      if (c.status == 4) {
        add(gi, "no contacts");
        continue;
      }
      for (int ci = 0; ci < c.n_contacts; ++ci) {
        if (c.contact_state[ci] == 1) {
          add(gi, "contact with invalid link id");
          continue;
        }
        if (c.contact_state[ci] == 2) {
          add(gi, "contact normal not unit length");
          continue;
        }
        if (c.hand_dist[ci] > p->contact_tol)
          add(gi, "contact " + std::to_string(ci) + " is " + num(c.hand_dist[ci]) +
                      " m off the hand surface (limit " + num(p->contact_tol) + ")");
        if (c.object_dist[ci] > p->contact_tol)
          add(gi, "contact " + std::to_string(ci) + " is " + num(c.object_dist[ci]) +
                      " m off the object surface (limit " + num(p->contact_tol) + ")");
      }
      if (c.worst_depth > p->penetration_margin)
        add(gi, "object penetrates the hand by " + num(c.worst_depth) + " m (limit " +
                    num(p->penetration_margin) + ")");
      if (c.wrench_error == 1) {
        add(gi, "wrench recheck failed: tangent_basis: zero normal");
      } else if (c.wrench_error == 2) {
        add(gi, "wrench recheck failed: tangent_basis: normal is not unit length");
      } else if (!(c.wrench_objective < p->eps_stable)) {
        add(gi, "wrench objective " + num(c.wrench_objective) + " not under stability threshold " +
                    num(p->eps_stable));
      }
    }
    if (needed) *needed = out.size() + 1;
    if (n_issues) *n_issues = count;
    if (buf && cap) {
      size_t m = std::min(cap - 1, out.size());
      std::memcpy(buf, out.data(), m);
      buf[m] = '\0';
    }
  });
}

}  // extern "C"
