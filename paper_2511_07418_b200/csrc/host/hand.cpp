// hand.cpp — URDF-subset hand loader (reference hand.cpp:265-414), parts
// manifest, dependency groups (hand.cpp:515-552) and the host steps of
// build_field: per-link surface sampling + patch decomposition
// (pipeline.cpp:277-285, contact_field.cpp:26-99).  The reference parses
// XML with Boost.PropertyTree and JSON with nlohmann; neither exists in this
// image, so a minimal parser for exactly the subset the loader reads lives
// here.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <map>
#include <random>
#include <sstream>
#include <stdexcept>

#include "host.hpp"

namespace lgh {

using namespace lgm;

namespace {

// ------------------------------------------------------------ mini XML
struct XNode {
  std::string name;
  std::vector<std::pair<std::string, std::string>> attrs;
  std::vector<XNode> kids;
  const XNode* child(const std::string& n) const {
    for (const auto& k : kids)
      if (k.name == n) return &k;
    return nullptr;
  }
  const std::string* attr(const std::string& n) const {
    for (const auto& a : attrs)
      if (a.first == n) return &a.second;
    return nullptr;
  }
};

struct XParser {
  const std::string& s;
  size_t i = 0;
  explicit XParser(const std::string& src) : s(src) {}
  [[noreturn]] void bad(const std::string& w) {
    throw std::runtime_error("xml: " + w + " at offset " + std::to_string(i));
  }
  void ws() {
    while (i < s.size() && std::isspace((unsigned char)s[i])) ++i;
  }
  bool starts(const char* t) { return s.compare(i, std::strlen(t), t) == 0; }
  void skip_misc() {
    for (;;) {
      ws();
      if (starts("<?")) {
        size_t e = s.find("?>", i);
        if (e == std::string::npos) bad("unterminated declaration");
        i = e + 2;
      } else if (starts("<!--")) {
        size_t e = s.find("-->", i);
        if (e == std::string::npos) bad("unterminated comment");
        i = e + 3;
      } else if (starts("<!")) {
        size_t e = s.find('>', i);
        if (e == std::string::npos) bad("unterminated directive");
        i = e + 1;
      } else {
        return;
      }
    }
  }
  static std::string unescape(const std::string& v) {
    std::string o;
    for (size_t k = 0; k < v.size(); ++k) {
      if (v[k] == '&') {
        size_t e = v.find(';', k);
        if (e != std::string::npos) {
          std::string ent = v.substr(k + 1, e - k - 1);
          const char* rep = ent == "lt" ? "<" : ent == "gt" ? ">" : ent == "amp" ? "&"
                            : ent == "quot" ? "\"" : ent == "apos" ? "'" : nullptr;
          if (rep) {
            o += rep;
            k = e;
            continue;
          }
        }
      }
      o += v[k];
    }
    return o;
  }
  std::string name() {
    size_t b = i;
    while (i < s.size() && !std::isspace((unsigned char)s[i]) && s[i] != '>' && s[i] != '/' &&
           s[i] != '=')
      ++i;
    if (b == i) bad("expected a name");
    return s.substr(b, i - b);
  }
  XNode element() {
    if (i >= s.size() || s[i] != '<') bad("expected '<'");
    ++i;
    XNode n;
    n.name = name();
    for (;;) {
      ws();
      if (i >= s.size()) bad("unexpected end");
      if (s[i] == '/') {
        if (i + 1 >= s.size() || s[i + 1] != '>') bad("expected '/>'");
        i += 2;
        return n;
      }
      if (s[i] == '>') {
        ++i;
        break;
      }
      std::string an = name();
      ws();
      if (i >= s.size() || s[i] != '=') bad("expected '='");
      ++i;
      ws();
      char q = s[i];
      if (q != '"' && q != '\'') bad("expected quote");
      size_t e = s.find(q, i + 1);
      if (e == std::string::npos) bad("unterminated attribute");
      n.attrs.push_back({an, unescape(s.substr(i + 1, e - i - 1))});
      i = e + 1;
    }
    for (;;) {
      // text content is ignored by the loader
      while (i < s.size() && s[i] != '<') ++i;
      if (i >= s.size()) bad("unterminated element " + n.name);
      if (starts("<!--")) {
        size_t e = s.find("-->", i);
        if (e == std::string::npos) bad("unterminated comment");
        i = e + 3;
        continue;
      }
      if (starts("</")) {
        i += 2;
        std::string cn = name();
        if (cn != n.name) bad("mismatched </" + cn + ">");
        ws();
        if (i >= s.size() || s[i] != '>') bad("expected '>'");
        ++i;
        return n;
      }
      n.kids.push_back(element());
    }
  }
};

// ------------------------------------------------------------ mini JSON
// parts manifest: {"link": ["file", ...], ...}; keys iterate sorted (the
// nlohmann::json object is a std::map).
std::map<std::string, std::vector<std::string>> parse_manifest(const std::string& s) {
  size_t i = 0;
  auto ws = [&]() {
    while (i < s.size() && std::isspace((unsigned char)s[i])) ++i;
  };
  auto bad = [&](const char* w) -> void {
    throw std::runtime_error(std::string("parts manifest: ") + w);
  };
  auto str = [&]() {
    ws();
    if (i >= s.size() || s[i] != '"') bad("expected string");
    std::string o;
    ++i;
    while (i < s.size() && s[i] != '"') {
      if (s[i] == '\\' && i + 1 < s.size()) ++i;
      o += s[i++];
    }
    if (i >= s.size()) bad("unterminated string");
    ++i;
    return o;
  };
  std::map<std::string, std::vector<std::string>> out;
  ws();
  if (i >= s.size() || s[i] != '{') bad("expected object");
  ++i;
  ws();
  if (i < s.size() && s[i] == '}') return out;
  for (;;) {
    std::string key = str();
    ws();
    if (i >= s.size() || s[i] != ':') bad("expected ':'");
    ++i;
    ws();
    if (i >= s.size() || s[i] != '[') bad("expected array");
    ++i;
    std::vector<std::string> files;
    ws();
    if (i < s.size() && s[i] == ']') {
      ++i;
    } else {
      for (;;) {
        files.push_back(str());
        ws();
        if (i < s.size() && s[i] == ',') {
          ++i;
          continue;
        }
        if (i < s.size() && s[i] == ']') {
          ++i;
          break;
        }
        bad("expected ',' or ']'");
      }
    }
    out[key] = files;
    ws();
    if (i < s.size() && s[i] == ',') {
      ++i;
      continue;
    }
    if (i < s.size() && s[i] == '}') break;
    bad("expected ',' or '}'");
  }
  return out;
}

V3 parse_vec3(const std::string& text, const char* what) {  // hand.cpp:196-204
  std::istringstream ss(text);
  double x, y, z;
  ss >> x >> y >> z;
  if (ss.fail()) throw std::runtime_error(std::string("bad ") + what + ": " + text);
  return v3(x, y, z);
}

double parse_double(const std::string& text, const char* what) {
  std::istringstream ss(text);
  double v;
  ss >> v;
  if (ss.fail()) throw std::runtime_error(std::string("bad ") + what + ": " + text);
  return v;
}

const std::string& req_attr(const XNode& n, const char* a) {
  const std::string* v = n.attr(a);
  if (!v) throw std::runtime_error(std::string("hand file: <") + n.name + "> needs " + a);
  return *v;
}

// Eigen quaternion product (w, x, y, z)
void qmul(const double* a, const double* b, double* o) {
  o[0] = a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3];
  o[1] = a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2];
  o[2] = a[0] * b[2] + a[2] * b[0] + a[3] * b[1] - a[1] * b[3];
  o[3] = a[0] * b[3] + a[3] * b[0] + a[1] * b[2] - a[2] * b[1];
}

// URDF rpy: Rz(yaw) Ry(pitch) Rx(roll) as an Eigen AngleAxis product
// (hand.cpp:206-220), glibc trig.
Xf parse_origin(const XNode& node) {
  Xf t = xf_identity();
  const XNode* o = node.child("origin");
  if (!o) return t;
  const std::string* xyz = o->attr("xyz");
  const std::string* rpy = o->attr("rpy");
  t.t = parse_vec3(xyz ? *xyz : "0 0 0", "origin xyz");
  V3 r = parse_vec3(rpy ? *rpy : "0 0 0", "origin rpy");
  // AngleAxis -> Quaternion: w = cos(a/2), vec = sin(a/2) * axis
  double sz = std::sin(0.5 * r.z), sy = std::sin(0.5 * r.y), sx = std::sin(0.5 * r.x);
  double qz[4] = {std::cos(0.5 * r.z), sz * 0.0, sz * 0.0, sz * 1.0};
  double qy[4] = {std::cos(0.5 * r.y), sy * 0.0, sy * 1.0, sy * 0.0};
  double qx[4] = {std::cos(0.5 * r.x), sx * 1.0, sx * 0.0, sx * 0.0};
  double a[4], q[4];
  qmul(qz, qy, a);
  qmul(a, qx, q);
  t.R = quat_to_matrix(q[0], q[1], q[2], q[3]);
  return t;
}

Mesh parse_geometry(const XNode& geom, const std::string& base) {  // hand.cpp:227-252
  if (const XNode* m = geom.child("mesh")) {
    Mesh mesh = load_mesh(base + "/" + req_attr(*m, "filename"));
    const std::string* sc = m->attr("scale");
    V3 s = parse_vec3(sc ? *sc : "1 1 1", "mesh scale");
    if (!(s.x == 1.0 && s.y == 1.0 && s.z == 1.0))
      for (V3& v : mesh.verts) v = cmul(v, s);
    return mesh;
  }
  if (const XNode* b = geom.child("box")) return make_box(parse_vec3(req_attr(*b, "size"), "box size"), v3(0, 0, 0));
  if (const XNode* s = geom.child("sphere"))
    return make_icosphere(parse_double(req_attr(*s, "radius"), "radius"), 2, v3(0, 0, 0));
  if (const XNode* c = geom.child("cylinder"))
    return make_cylinder(parse_double(req_attr(*c, "radius"), "radius"),
                         parse_double(req_attr(*c, "length"), "length"), 24);
  throw std::runtime_error("unsupported geometry element in hand file");
}

std::string read_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open " + path);
  std::stringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

}  // namespace

int Hand::link_index(const std::string& n) const {
  for (size_t i = 0; i < links.size(); ++i)
    if (links[i].name == n) return (int)i;
  return -1;
}

Hand load_hand(const std::string& path, double scale_) {  // hand.cpp:265-414
  XNode doc;
  try {
    std::string src = read_file(path);
    XParser p(src);
    p.skip_misc();
    doc = p.element();
  } catch (const std::exception& e) {
    throw std::runtime_error("cannot parse hand file " + path + ": " + e.what());
  }
  if (doc.name != "robot") throw std::runtime_error("hand file has no <robot> element");
  Hand h;
  auto slash = path.find_last_of('/');
  h.source_dir = slash == std::string::npos ? std::string(".") : path.substr(0, slash);
  for (const XNode& node : doc.kids) {
    if (node.name != "link") continue;
    Link link;
    link.name = req_attr(node, "name");
    if (h.link_index(link.name) >= 0) throw std::runtime_error("duplicate link name: " + link.name);
    for (const XNode& ch : node.kids) {
      if (ch.name != "visual") continue;
      Xf vo = parse_origin(ch);
      const XNode* g = ch.child("geometry");
      if (!g) throw std::runtime_error("visual without geometry");
      Mesh m = parse_geometry(*g, h.source_dir);
      int base = (int)link.visual.verts.size();
      for (const V3& v : m.verts) link.visual.verts.push_back(xf_apply(vo, v));
      for (const auto& t : m.tris) link.visual.tris.push_back({t[0] + base, t[1] + base, t[2] + base});
    }
    h.links.push_back(std::move(link));
  }
  if (h.links.empty()) throw std::runtime_error("hand file has no links");
  int joints = 0;
  for (const XNode& node : doc.kids) {
    if (node.name != "joint") continue;
    std::string type = req_attr(node, "type");
    std::string name = req_attr(node, "name");
    const XNode* pn = node.child("parent");
    const XNode* cn = node.child("child");
    int parent = pn ? h.link_index(req_attr(*pn, "link")) : -1;
    int child = cn ? h.link_index(req_attr(*cn, "link")) : -1;
    if (parent < 0 || child < 0) throw std::runtime_error("joint " + name + " references unknown link");
    Link& cl = h.links[child];
    if (cl.parent >= 0) throw std::runtime_error("link " + cl.name + " has two parent joints");
    cl.parent = parent;
    cl.joint_name = name;
    cl.origin = parse_origin(node);
    if (type == "fixed") {
      cl.jtype = 0;
    } else if (type == "revolute" || type == "prismatic") {
      cl.jtype = type == "revolute" ? 1 : 2;
      const XNode* ax = node.child("axis");
      const std::string* axs = ax ? ax->attr("xyz") : nullptr;
      cl.axis = parse_vec3(axs ? *axs : "1 0 0", "joint axis");
      double len = norm(cl.axis);
      if (len < 1e-9) throw std::runtime_error("joint " + name + ": zero axis");
      cl.axis = divs(cl.axis, len);
      const XNode* lim = node.child("limit");
      if (!lim) throw std::runtime_error("joint " + name + " has no limit element");
      cl.lo = parse_double(req_attr(*lim, "lower"), "limit");
      cl.hi = parse_double(req_attr(*lim, "upper"), "limit");
      if (cl.lo > cl.hi) throw std::runtime_error("joint " + name + ": lower limit above upper");
      cl.jidx = joints++;
    } else {
      throw std::runtime_error("unsupported joint type '" + type + "' on " + name);
    }
  }
  h.dof = joints;
  for (size_t i = 0; i < h.links.size(); ++i) {
    if (h.links[i].parent < 0) {
      if (h.root >= 0) throw std::runtime_error("hand file has multiple root links");
      h.root = (int)i;
    }
  }
  if (h.root < 0) throw std::runtime_error("hand file has no root link (cycle)");
  std::vector<std::vector<int>> children(h.links.size());
  for (size_t i = 0; i < h.links.size(); ++i)
    if (h.links[i].parent >= 0) children[h.links[i].parent].push_back((int)i);
  std::vector<int> stack = {h.root};
  while (!stack.empty()) {
    int l = stack.back();
    stack.pop_back();
    h.topo.push_back(l);
    for (auto it = children[l].rbegin(); it != children[l].rend(); ++it) stack.push_back(*it);
    if (h.topo.size() > h.links.size()) break;
  }
  if (h.topo.size() != h.links.size()) throw std::runtime_error("hand kinematic graph is not a tree");

  std::string stem = path;
  auto dot = stem.rfind('.');
  if (dot != std::string::npos) stem = stem.substr(0, dot);
  std::ifstream manifest(stem + ".parts.json");
  if (manifest) {
    std::stringstream ss;
    ss << manifest.rdbuf();
    for (const auto& kv : parse_manifest(ss.str())) {
      int l = h.link_index(kv.first);
      if (l < 0) throw std::runtime_error("parts manifest references unknown link " + kv.first);
      for (const auto& f : kv.second)
        h.links[l].parts.push_back(convex_hull(load_mesh(h.source_dir + "/" + f).verts));
    }
  } else {
    for (auto& link : h.links)
      if (link.visual.verts.size() >= 4) link.parts.push_back(convex_hull(link.visual.verts));
  }
  if (scale_ != 1.0) {
    if (scale_ <= 0.0) throw std::runtime_error("hand scale must be positive");
    for (auto& link : h.links) {
      link.origin.t = scale(scale_, link.origin.t);
      for (V3& v : link.visual.verts) v = scale(scale_, v);
      for (auto& part : link.parts) part = scale_part(part, scale_);
      if (link.jtype == 2) {
        link.lo *= scale_;
        link.hi *= scale_;
      }
    }
  }
  h.flatten();
  return h;
}

void Hand::flatten() {
  int n = (int)links.size();
  f_parent.assign(n, -1);
  f_jtype.assign(n, 0);
  f_jidx.assign(n, -1);
  f_R.assign(9 * n, 0.0);
  f_t.assign(3 * n, 0.0);
  f_axis.assign(3 * n, 0.0);
  f_lo.assign(n, 0.0);
  f_hi.assign(n, 0.0);
  f_part_link.clear();
  f_vert_off = {0};
  f_tri_off = {0};
  f_plane_off = {0};
  f_verts.clear();
  f_tris.clear();
  f_planes.clear();
  f_bounds.clear();
  for (int l = 0; l < n; ++l) {
    const Link& k = links[l];
    f_parent[l] = k.parent;
    f_jtype[l] = k.jtype;
    f_jidx[l] = k.jidx;
    m3_store(&f_R[9 * l], k.origin.R);
    v3_store(&f_t[3 * l], k.origin.t);
    v3_store(&f_axis[3 * l], k.axis);
    f_lo[l] = k.lo;
    f_hi[l] = k.hi;
    for (const Part& p : k.parts) {
      f_part_link.push_back(l);
      for (const V3& v : p.verts) f_verts.insert(f_verts.end(), {v.x, v.y, v.z});
      for (const auto& t : p.tris) f_tris.insert(f_tris.end(), {t[0], t[1], t[2]});
      for (size_t i = 0; i < p.plane_n.size(); ++i)
        f_planes.insert(f_planes.end(), {p.plane_n[i].x, p.plane_n[i].y, p.plane_n[i].z, p.plane_d[i]});
      f_bounds.insert(f_bounds.end(), {p.bmin.x, p.bmin.y, p.bmin.z, p.bmax.x, p.bmax.y, p.bmax.z});
      f_vert_off.push_back((int)(f_verts.size() / 3));
      f_tri_off.push_back((int)(f_tris.size() / 3));
      f_plane_off.push_back((int)(f_planes.size() / 4));
    }
  }
}

lg_hand_desc Hand::desc() const {
  lg_hand_desc d;
  std::memset(&d, 0, sizeof(d));
  d.n_links = (int)links.size();
  d.dof = dof;
  d.root = root;
  d.parent = f_parent.data();
  d.joint_type = f_jtype.data();
  d.joint_index = f_jidx.data();
  d.topo_order = topo.data();
  d.origin_R = f_R.data();
  d.origin_t = f_t.data();
  d.axis = f_axis.data();
  d.limit_lo = f_lo.data();
  d.limit_hi = f_hi.data();
  d.n_parts = (int)f_part_link.size();
  d.part_link = f_part_link.data();
  d.part_vert_off = f_vert_off.data();
  d.part_verts = f_verts.data();
  d.part_tri_off = f_tri_off.data();
  d.part_tris = f_tris.data();
  d.part_plane_off = f_plane_off.data();
  d.part_planes = f_planes.data();
  d.part_bounds = f_bounds.data();
  return d;
}

std::vector<int> dependency_group_of(const Hand& h, int* n_groups) {  // hand.cpp:515-552
  int n = (int)h.links.size();
  std::vector<bool> is_static(n, false);
  for (int l : h.topo) {
    const Link& k = h.links[l];
    if (k.parent < 0) is_static[l] = true;
    else if (is_static[k.parent] && k.jtype == 0) is_static[l] = true;
  }
  std::vector<int> seed_of(n, -1);
  std::map<int, std::vector<int>> by_seed;
  for (int l : h.topo) {
    if (is_static[l]) continue;
    int p = h.links[l].parent;
    seed_of[l] = (p >= 0 && !is_static[p]) ? seed_of[p] : l;
    by_seed[seed_of[l]].push_back(l);
  }
  std::vector<std::vector<int>> groups;
  for (auto& kv : by_seed) {
    std::sort(kv.second.begin(), kv.second.end());
    groups.push_back(kv.second);
  }
  std::sort(groups.begin(), groups.end(),
            [](const std::vector<int>& a, const std::vector<int>& b) { return a[0] < b[0]; });
  std::vector<int> out(n, -1);
  for (size_t g = 0; g < groups.size(); ++g)
    for (int l : groups[g]) out[l] = (int)g;
  if (n_groups) *n_groups = (int)groups.size();
  return out;
}

lg_patches_desc Patches::desc() const {
  lg_patches_desc d;
  d.n_patches = (int)link.size();
  d.link = link.data();
  d.point_off = point_off.data();
  d.points = pts.data();
  d.normals = nrm.data();
  d.fp_off = fp_off.data();
  d.field_points = fps.data();
  return d;
}

Patches make_patches(const Hand& h, double spc, double radius, uint64_t seed, int cap) {
  const uint64_t kTagHandSamples = 0x686e6473;  // pipeline.cpp:20
  const uint64_t kTagPatch = 0x70617463;        // contact_field.cpp:16
  const uint64_t kTagSubset = 0x73756273;       // contact_field.cpp:17
  std::vector<std::vector<Sample>> per(h.links.size());
  size_t total = 0;
  for (size_t l = 0; l < h.links.size(); ++l) {
    if (h.links[l].visual.verts.empty()) continue;
    per[l] = sample_surface(h.links[l].visual, spc, mix_seed(seed, kTagHandSamples, l));
    total += per[l].size();
  }
  if (radius <= 0.0 || cap < 1) fail_invalid("decompose_patches: bad radius or cap");
  if (total == 0) fail_invalid("decompose_patches: no surface samples");
  const double gather = 0.5 * radius;
  Patches P;
  P.point_off.push_back(0);
  P.fp_off.push_back(0);
  int next_id = 0;
  for (size_t link = 0; link < per.size(); ++link) {
    const auto& S = per[link];
    if (S.empty()) continue;
    std::mt19937_64 rng(mix_seed(seed, kTagPatch, link));
    std::vector<int> uncovered(S.size());
    for (size_t i = 0; i < S.size(); ++i) uncovered[i] = (int)i;
    while (!uncovered.empty()) {
      size_t pick = rng() % uncovered.size();
      int sid = uncovered[pick];
      V3 center = S[sid].p;
      std::vector<V3> pts = {center}, nrm = {S[sid].n};
      std::vector<int> rest;
      for (int id : uncovered) {
        if (id == sid) continue;
        if (norm(sub(S[id].p, center)) <= gather) {
          pts.push_back(S[id].p);
          nrm.push_back(S[id].n);
        } else {
          rest.push_back(id);
        }
      }
      uncovered.swap(rest);
      int id = next_id++;
      int m = (int)pts.size();
      std::vector<int> fp;
      if (m <= cap) {
        for (int i = 0; i < m; ++i) fp.push_back(i);
      } else {
        std::mt19937_64 sr(mix_seed(seed, kTagSubset, (uint64_t)id));
        std::vector<int> pool(m - 1);
        for (int i = 1; i < m; ++i) pool[i - 1] = i;
        fp.push_back(0);
        for (int i = 0; i < cap - 1; ++i) {
          size_t j = i + sr() % (pool.size() - i);
          std::swap(pool[i], pool[j]);
          fp.push_back(pool[i]);
        }
        std::sort(fp.begin(), fp.end());
      }
      P.link.push_back((int)link);
      for (int i = 0; i < m; ++i) {
        P.pts.insert(P.pts.end(), {pts[i].x, pts[i].y, pts[i].z});
        P.nrm.insert(P.nrm.end(), {nrm[i].x, nrm[i].y, nrm[i].z});
      }
      P.point_off.push_back((int)(P.pts.size() / 3));
      P.fps.insert(P.fps.end(), fp.begin(), fp.end());
      P.fp_off.push_back((int)P.fps.size());
    }
  }
  return P;
}

}  // namespace lgh
