// lg_device.cu — device half of the C-ABI: context, contact-field build,
// batched stage entry points and the run_batch driver (reference
// pipeline.cpp:308-625) on one B200.  Single translation unit so that the
// constant-memory hand model is visible to every kernel.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <filesystem>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include <cub/device/device_segmented_sort.cuh>

#include "../capi_common.hpp"
#include "dev_copt.cuh"
#include "dev_post.cuh"
#include "dev_validate.cuh"
#include "dev_patches.cuh"

using namespace lgd;

namespace {

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess)                                                             \
      throw lgc::cuda_error(std::string(#x) + ": " + cudaGetErrorString(e_));          \
  } while (0)

// ---------------------------------------------------------------- buffers
// Device scratch comes from cudaMalloc through a per-stream block cache: a
// pass allocates the same buffer sizes every call, so released blocks are
// kept and handed back (stream order makes reuse on the same stream safe).
// The cache of a stream is bounded (kCacheCap bytes; the largest blocks are
// returned to the driver first) and is dropped entirely, then the allocation
// retried once, when cudaMalloc reports out-of-memory.
thread_local cudaStream_t g_alloc_stream = nullptr;
std::mutex g_streams_mu;
std::set<cudaStream_t> g_live_streams;  // streams of live contexts
std::map<cudaStream_t, std::multimap<size_t, void*>> g_cache;
std::map<cudaStream_t, size_t> g_cache_bytes;
constexpr size_t kCacheCap = size_t(64) << 30;  // of 180 GB HBM

void drop_cache(cudaStream_t s);

// cudaMalloc calls and their host time (LG_TIMING reports them per call)
thread_local long long g_malloc_calls = 0;
thread_local double g_malloc_ms = 0.0;

void* cached_alloc(size_t bytes, cudaStream_t s) {
  {
    std::lock_guard<std::mutex> lk(g_streams_mu);
    if (g_live_streams.count(s)) {
      auto& c = g_cache[s];
      // best fit within 1/8: a request does not take a much larger block
      // that a later, larger request of the same call needs (the pass makes
      // the same requests every call, so the cache then settles after one
      // call; each cudaMalloc costs milliseconds here)
      auto it = c.lower_bound(bytes);
      if (it != c.end() && it->first <= bytes + bytes / 8 + 4096) {
        void* p = it->second;
        g_cache_bytes[s] -= it->first;
        c.erase(it);
        return p;
      }
    }
  }
  void* p = nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  cudaError_t e = cudaMalloc(&p, bytes);
  g_malloc_calls += 1;
  g_malloc_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  if (e == cudaErrorMemoryAllocation) {
    (void)cudaGetLastError();
    CK(cudaStreamSynchronize(s));
    drop_cache(s);
    e = cudaMalloc(&p, bytes);
  }
  CK(e);
  return p;
}

void free_on(void* p, size_t bytes, cudaStream_t s) {
  {
    std::lock_guard<std::mutex> lk(g_streams_mu);
    if (g_live_streams.count(s)) {
      auto& c = g_cache[s];
      size_t& held = g_cache_bytes[s];
      c.emplace(bytes, p);
      held += bytes;
      // bounded: return the largest blocks to the driver first
      while (held > kCacheCap && !c.empty()) {
        auto last = std::prev(c.end());
        held -= last->first;
        cudaFree(last->second);
        c.erase(last);
      }
      return;
    }
  }
  // a buffer that outlives its context (e.g. a field destroyed after the
  // context) is freed synchronously
  cudaFree(p);
}

void drop_cache(cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_streams_mu);
  auto it = g_cache.find(s);
  if (it == g_cache.end()) return;
  for (auto& kv : it->second) cudaFree(kv.second);
  g_cache.erase(it);
  g_cache_bytes.erase(s);
}

// Canary mode (LG_CHECK_CANARY=1, read once): every device buffer gets a
// 4 KiB guard band after the requested bytes, filled with 0xA5 at allocation
// and verified at release; a kernel writing past the end of any buffer is
// counted (lg_debug_canary_violations) and reported on stderr.  The device
// substitute for compute-sanitizer's out-of-bounds-write check, which this
// GPU pool does not allow.
constexpr size_t kGuard = 4096;
bool canary_on() {
  static const bool on = [] {
    const char* e = std::getenv("LG_CHECK_CANARY");
    return e && e[0] == '1';
  }();
  return on;
}
std::atomic<long long> g_canary_bad{0};

struct Buf {
  void* p = nullptr;
  size_t n = 0;
  size_t req = 0;  // requested bytes (canary mode: the guard starts here)
  cudaStream_t s = nullptr;
  Buf() = default;
  Buf(const Buf&) = delete;
  Buf& operator=(const Buf&) = delete;
  ~Buf() { release(); }
  void check_guard() {
    if (!p || !canary_on()) return;
    std::vector<unsigned char> g(n - req);
    if (cudaStreamSynchronize(s) != cudaSuccess ||
        cudaMemcpy(g.data(), (char*)p + req, g.size(), cudaMemcpyDeviceToHost) != cudaSuccess)
      return;
    for (unsigned char c : g)
      if (c != 0xA5) {
        ++g_canary_bad;
        std::fprintf(stderr, "lg: canary: write past the end of a %zu-byte device buffer\n", req);
        return;
      }
  }
  void release() {
    check_guard();
    if (p) free_on(p, n, s);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t bytes) {
    if (bytes <= n && p && !canary_on()) return;
    if (p) release();
    req = bytes;
    bytes = (bytes + 255) & ~(size_t)255;
    if (bytes == 0) bytes = 256;
    if (canary_on()) bytes += kGuard;
    s = g_alloc_stream;
    p = cached_alloc(bytes, s);
    n = bytes;
    if (canary_on()) CK(cudaMemsetAsync((char*)p + req, 0xA5, n - req, s));
  }
  template <typename T>
  T* as() const {
    return (T*)p;
  }
};

template <typename T>
T* dalloc(Buf& b, size_t count) {
  b.alloc(count * sizeof(T));
  return b.as<T>();
}
// PCIe traffic accounting (reported as h2d_bytes / d2h_bytes per run)
// PCIe bytes moved by the current call, per host thread (one in-flight call
// per context, one context per driving thread).
thread_local long long g_h2d = 0, g_d2h = 0;

template <typename T>
T* dupload(Buf& b, const T* src, size_t count, cudaStream_t s) {
  T* d = dalloc<T>(b, count);
  if (count) CK(cudaMemcpyAsync(d, src, count * sizeof(T), cudaMemcpyHostToDevice, s));
  g_h2d += (long long)(count * sizeof(T));
  return d;
}
template <typename T>
std::vector<T> ddownload(const T* src, size_t count, cudaStream_t s) {
  std::vector<T> v(count);
  g_d2h += (long long)(count * sizeof(T));
  if (count) CK(cudaMemcpyAsync(v.data(), src, count * sizeof(T), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return v;
}

int grid_for(long long n, int block) {
  long long g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > 148 * 64) g = 148 * 64;
  return (int)g;
}

int bits_for(unsigned long long range) {
  int b = 0;
  while (b < 64 && (range >> b) != 0ull) ++b;
  return b;
}

// Host-side dependency groups from a flat description (hand.cpp:374-411).
std::vector<int> groups_of(const lg_hand_desc& h, int* n_groups) {
  int n = h.n_links;
  std::vector<bool> st(n, false);
  for (int ii = 0; ii < n; ++ii) {
    int l = h.topo_order[ii];
    if (h.parent[l] < 0) st[l] = true;
    else if (st[h.parent[l]] && h.joint_type[l] == 0) st[l] = true;
  }
  std::vector<int> seed(n, -1);
  std::map<int, std::vector<int>> by;
  for (int ii = 0; ii < n; ++ii) {
    int l = h.topo_order[ii];
    if (st[l]) continue;
    int p = h.parent[l];
    seed[l] = (p >= 0 && !st[p]) ? seed[p] : l;
    by[seed[l]].push_back(l);
  }
  std::vector<std::vector<int>> groups;
  for (auto& kv : by) {
    std::sort(kv.second.begin(), kv.second.end());
    groups.push_back(kv.second);
  }
  std::sort(groups.begin(), groups.end(),
            [](const std::vector<int>& a, const std::vector<int>& b) { return a[0] < b[0]; });
  std::vector<int> out(n, -1);
  for (size_t g = 0; g < groups.size(); ++g)
    for (int l : groups[g]) out[l] = (int)g;
  *n_groups = (int)groups.size();
  return out;
}

std::vector<double> make_codebook(int size) {  // contact_field.cpp:144-158 (host, glibc)
  if (size < 1 || size > 65536) throw std::invalid_argument("make_codebook: size out of range");
  std::vector<double> d(3 * size);
  const double kPiH = 3.14159265358979323846;
  const double golden = kPiH * (3.0 - std::sqrt(5.0));
  for (int i = 0; i < size; ++i) {
    double z = 1.0 - 2.0 * (i + 0.5) / size;
    double r = std::sqrt(std::max(0.0, 1.0 - z * z));
    double a = golden * i;
    d[3 * i] = r * std::cos(a);
    d[3 * i + 1] = r * std::sin(a);
    d[3 * i + 2] = z;
  }
  return d;
}

}  // namespace

// ------------------------------------------------------------------ ctx
struct lg_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  void* cub_tmp = nullptr;
  size_t cub_n = 0;
  // hand currently bound to constant memory
  Buf h_vert_off, h_verts, h_tri_off, h_tris, h_plane_off, h_planes, h_bounds, h_part_link;
  int n_parts = 0;
  long long launches = 0;
  void* tmp(size_t n) {
    if (n > cub_n) {
      if (cub_tmp) cudaFree(cub_tmp);
      cub_tmp = nullptr;
      CK(cudaMalloc(&cub_tmp, n));
      cub_n = n;
    }
    return cub_tmp;
  }
};

namespace {

void use_ctx(lg_ctx* ctx) {
  CK(cudaSetDevice(ctx->device));
  g_alloc_stream = ctx->stream;
}

#define LAUNCH(ctx) ++(ctx)->launches

void check_launch() { CK(cudaGetLastError()); }

// Dynamic shared memory for a query kernel's codebook copy ([C][3] doubles),
// or 0 to read it from global memory: opts the kernel in above the default
// 48 KiB when needed, within the device's per-block limit minus the kernel's
// static shared memory.
template <typename K>
size_t codebook_smem(K kern, int C) {
  const size_t need = 3 * (size_t)C * sizeof(double);
  cudaFuncAttributes a;
  CK(cudaFuncGetAttributes(&a, kern));
  int dev = 0, optin = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  if (need + a.sharedSizeBytes > (size_t)optin || need > (size_t)(64 << 10)) return 0;
  if (need > (size_t)a.maxDynamicSharedSizeBytes)
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need));
  return need;
}

// Binds a hand description to constant memory (one hand per call).
void bind_hand(lg_ctx* ctx, const lg_hand_desc& d) {
  if (d.n_links > kMaxLinks) throw std::invalid_argument("device: hand has too many links (max 32)");
  if (d.dof > kMaxDof) throw std::invalid_argument("device: hand has too many joints (max 24)");
  if (d.n_parts > 63) throw std::invalid_argument("device: hand has too many convex parts (max 63)");
  DHand h;
  std::memset(&h, 0, sizeof(h));
  h.n_links = d.n_links;
  h.dof = d.dof;
  h.root = d.root;
  h.n_parts = d.n_parts;
  for (int l = 0; l < d.n_links; ++l) {
    h.parent[l] = d.parent[l];
    h.jtype[l] = d.joint_type[l];
    h.jidx[l] = d.joint_index[l];
    h.topo[l] = d.topo_order[l];
    for (int a = 0; a < 9; ++a) h.R[l][a] = d.origin_R[9 * l + a];
    for (int a = 0; a < 3; ++a) {
      h.t[l][a] = d.origin_t[3 * l + a];
      h.axis[l][a] = d.axis[3 * l + a];
    }
    h.lo[l] = d.limit_lo[l];
    h.hi[l] = d.limit_hi[l];
    h.part_begin[l] = 0;
    h.part_end[l] = 0;
    if (d.joint_index[l] >= 0) {
      h.jlo[d.joint_index[l]] = d.limit_lo[l];
      h.jhi[d.joint_index[l]] = d.limit_hi[l];
      h.mid[d.joint_index[l]] = 0.5 * (d.limit_lo[l] + d.limit_hi[l]);
    }
  }
  for (int l = 0; l < d.n_links; ++l) {
    int path[kMaxLinks + 1], n = 0;
    for (int x = l; x >= 0 && n <= kMaxLinks; x = d.parent[x]) path[n++] = x;
    if (n > kMaxDepth) throw std::invalid_argument("device: kinematic chain deeper than 10 links");
    h.chain_len[l] = n;
    h.level[l] = n - 1;
    h.n_levels = std::max(h.n_levels, n);
    h.jmask[l] = 0u;
    for (int i = 0; i < n; ++i) {
      int x = path[n - 1 - i];
      h.chain[l][i] = x;
      if (d.joint_index[x] >= 0) h.jmask[l] |= 1u << d.joint_index[x];
    }
    if (d.joint_index[l] >= 0) h.jlink[d.joint_index[l]] = l;
  }
  for (int p = 0; p < d.n_parts; ++p) {
    int l = d.part_link[p];
    if (p > 0 && d.part_link[p] < d.part_link[p - 1])
      throw std::invalid_argument("device: parts must be grouped by link");
    if (h.part_end[l] == 0) h.part_begin[l] = p;
    h.part_end[l] = p + 1;
  }
  cudaStream_t s = ctx->stream;
  int nv = d.n_parts ? d.part_vert_off[d.n_parts] : 0;
  int nt = d.n_parts ? d.part_tri_off[d.n_parts] : 0;
  int npl = d.n_parts ? d.part_plane_off[d.n_parts] : 0;
  static const int zero = 0;
  h.vert_off = dupload(ctx->h_vert_off, d.n_parts ? d.part_vert_off : &zero, d.n_parts + 1, s);
  h.verts = dupload(ctx->h_verts, d.part_verts, 3 * (size_t)nv, s);
  h.tri_off = dupload(ctx->h_tri_off, d.n_parts ? d.part_tri_off : &zero, d.n_parts + 1, s);
  h.tris = dupload(ctx->h_tris, d.part_tris, 3 * (size_t)nt, s);
  h.plane_off = dupload(ctx->h_plane_off, d.n_parts ? d.part_plane_off : &zero, d.n_parts + 1, s);
  h.planes = dupload(ctx->h_planes, d.part_planes, 4 * (size_t)npl, s);
  h.bounds = dupload(ctx->h_bounds, d.part_bounds, 6 * (size_t)d.n_parts, s);
  dupload(ctx->h_part_link, d.part_link, (size_t)d.n_parts, s);
  ctx->n_parts = d.n_parts;
  CK(cudaMemcpyToSymbolAsync(c_hand, &h, sizeof(DHand), 0, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyToSymbolAsync(g_hand, &h, sizeof(DHand), 0, cudaMemcpyHostToDevice, s));
}

// Kernel attributes are per device: set them the first time a (device,
// kernel family) pair is launched in this process.
bool first_on_device(int tag) {
  static std::mutex mu;
  static std::set<std::pair<int, int>> done;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  return done.insert({dev, tag}).second;
}

// realize_grasp, one warp per problem, 4 warps per CTA.
// k_collision3 instance: LG_COLL_MINB = 4 (128 registers), 5 (96) or 3 (160)
using CollKern = void (*)(int, CollCfg, const int*, const int*, const double*, const double*,
                          const double*, int, uint8_t*, double*);
CollKern coll_kernel(const CollCfg& c) {
  static const int minb = [] {
    const char* e = std::getenv("LG_COLL_MINB");
    int v = e ? std::atoi(e) : 4;
    return (v == 3 || v == 5) ? v : 4;
  }();
  if (c.grid.ok && c.raw.n >= kCollGridMin) return k_collision3<4, true>;
  return minb == 5 ? k_collision3<5, false> : (minb == 3 ? k_collision3<3, false> : k_collision3<4, false>);
}

void launch_realize_warp(cudaStream_t s, int n, int k, const int* kk, const IkCfg& P, int rounds,
                         int fine_iters, const double* tgt, int tgt_stride, const int* tl,
                         int tl_stride, const double* q_init, double* q_out, double* max_res,
                         int* finite, unsigned long long* used, int dof, int n_links,
                         const IkOut* ik_out = nullptr) {
  const int wpb = 4;
  const int kmax = kk ? kMaxK : k;
  size_t smem = realize_warp_smem(dof, kmax, n_links, wpb);
  static const int minb = [] {
    const char* e = std::getenv("LG_REALIZE_MINB");
    int v = e ? std::atoi(e) : 5;  // 5 CTAs/SM (96 regs) measured fastest
    return (v == 4 || v == 6) ? v : 5;
  }();
  if (first_on_device(1)) {
    CK(cudaFuncSetAttribute(k_realize_warp<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(k_realize_warp<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(k_realize_warp<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  }
  if (ik_out && first_on_device(17))
    CK(cudaFuncSetAttribute(k_realize_warp<4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            200 * 1024));
  auto kern = ik_out ? k_realize_warp<4, true>
                     : (minb == 6 ? k_realize_warp<6> : (minb == 5 ? k_realize_warp<5> : k_realize_warp<4>));
  // persistent grid: as many CTAs as fit at once (warps fetch problems)
  int dev = 0, sms = 0, per_sm = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * wpb, smem));
  const long long need = (n + wpb - 1) / wpb;
  const int grid = (int)std::max(1ll, std::min(need, (long long)std::max(1, per_sm) * sms));
  Buf bnext;
  int* d_next = dalloc<int>(bnext, 1);
  CK(cudaMemsetAsync(d_next, 0, sizeof(int), s));
  kern<<<grid, 32 * wpb, smem, s>>>(n, k, kk, kmax, P, rounds, fine_iters, tgt, tgt_stride, tl, tl_stride,
                                    q_init, q_out, max_res, finite, used, d_next,
                                    ik_out ? *ik_out : IkOut{});
}

// Flattened patch data on the device.
struct DevPatches {
  int P = 0, F = 0, npts = 0;
  Buf pts, nrm, link, point_off, fp_off, fps, fp_link, fp_point, fp_patch;
  std::vector<int> h_link, h_point_off, h_fp_off, h_fps;
  std::vector<double> h_pts, h_nrm;
};

void upload_patches(lg_ctx* ctx, const lg_patches_desc& d, DevPatches& o) {
  cudaStream_t s = ctx->stream;
  o.P = d.n_patches;
  if (o.P < 1) throw std::invalid_argument("index build: no patches");
  o.npts = d.point_off[o.P];
  o.F = d.fp_off[o.P];
  o.h_link.assign(d.link, d.link + o.P);
  o.h_point_off.assign(d.point_off, d.point_off + o.P + 1);
  o.h_fp_off.assign(d.fp_off, d.fp_off + o.P + 1);
  o.h_fps.assign(d.field_points, d.field_points + o.F);
  o.h_pts.assign(d.points, d.points + 3 * (size_t)o.npts);
  o.h_nrm.assign(d.normals, d.normals + 3 * (size_t)o.npts);
  std::vector<int> fl(o.F), fpnt(o.F), fpat(o.F);
  for (int p = 0; p < o.P; ++p)
    for (int f = d.fp_off[p]; f < d.fp_off[p + 1]; ++f) {
      fl[f] = d.link[p];
      fpnt[f] = d.point_off[p] + d.field_points[f];
      fpat[f] = p;
    }
  dupload(o.pts, d.points, 3 * (size_t)o.npts, s);
  dupload(o.nrm, d.normals, 3 * (size_t)o.npts, s);
  dupload(o.link, d.link, (size_t)o.P, s);
  dupload(o.point_off, d.point_off, (size_t)o.P + 1, s);
  dupload(o.fp_off, d.fp_off, (size_t)o.P + 1, s);
  dupload(o.fps, d.field_points, (size_t)o.F, s);
  dupload(o.fp_link, fl.data(), fl.size(), s);
  dupload(o.fp_point, fpnt.data(), fpnt.size(), s);
  dupload(o.fp_patch, fpat.data(), fpat.size(), s);
  CK(cudaStreamSynchronize(s));
}

}  // namespace

#include "dev_fieldbuild.cuh"

namespace {


// ------------------------------------------------------------- run_batch
struct RunOut {
  lg_profile profile;
  std::vector<lg_grasp> grasps;
  std::vector<lg_trace> traces;
};

struct Timer {
  cudaEvent_t a, b;
  cudaStream_t s;
  explicit Timer(cudaStream_t st) : s(st) {
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
  }
  ~Timer() {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
  void start() { CK(cudaEventRecord(a, s)); }
  double stop() {
    CK(cudaEventRecord(b, s));
    CK(cudaEventSynchronize(b));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, a, b));
    return ms * 1e-3;
  }
};

DSamples make_samples(Buf* cols, int n) {
  DSamples d;
  d.n = n;
  for (int a = 0; a < 6; ++a) d.x[a] = cols[a].as<double>();
  return d;
}

// Object sample grid (dev_stages.cuh DGrid) over the n samples S, whose host
// copy `host` is [n][6].  Cell width w (doubled until the grid has at most
// kGridMaxCells cells); ok = 0 (callers sweep every sample) when a sample
// coordinate is not finite.
struct GridBufs {
  Buf cnt, start, keys, keys2, vals, id, cols;
};
constexpr long long kGridMaxCells = 1ll << 22;
DGrid build_grid(lg_ctx* ctx, const DSamples& S, const double* host, int n, double w, GridBufs& gb,
                 cudaStream_t s) {
  DGrid g{};
  g.ok = 0;
  if (n <= 0 || !(w > 0.0) || !std::isfinite(w)) return g;
  double lo[3] = {kInf, kInf, kInf}, hi[3] = {-kInf, -kInf, -kInf};
  for (int i = 0; i < n; ++i)
    for (int a = 0; a < 3; ++a) {
      const double v = host[6 * i + a];
      if (!std::isfinite(v)) return g;
      lo[a] = std::min(lo[a], v);
      hi[a] = std::max(hi[a], v);
    }
  long long cells = 0;
  for (;;) {
    cells = 1;
    for (int a = 0; a < 3; ++a) {
      const double d = std::floor((hi[a] - lo[a]) / w) + 1.0;
      g.dim[a] = d > 2e6 ? 2000000 : (int)d;
      cells *= g.dim[a];
    }
    if (cells <= kGridMaxCells) break;
    w *= 2.0;
  }
  for (int a = 0; a < 3; ++a) g.lo[a] = lo[a];
  g.w = w;
  int* cnt = dalloc<int>(gb.cnt, (size_t)cells + 1);
  CK(cudaMemsetAsync(cnt, 0, sizeof(int) * ((size_t)cells + 1), s));
  unsigned* keys = dalloc<unsigned>(gb.keys, (size_t)n);
  unsigned* keys2 = dalloc<unsigned>(gb.keys2, (size_t)n);
  int* vals = dalloc<int>(gb.vals, (size_t)n);
  int* id = dalloc<int>(gb.id, (size_t)n);
  int* start = dalloc<int>(gb.start, (size_t)cells + 1);
  k_grid_keys<<<grid_for(n, 256), 256, 0, s>>>(S, g, keys, vals, cnt);
  LAUNCH(ctx);
  check_launch();
  size_t tb = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, start, (int)cells + 1, s));
  CK(cub::DeviceScan::ExclusiveSum(ctx->tmp(tb), tb, cnt, start, (int)cells + 1, s));
  LAUNCH(ctx);
  int bits = 1;
  while (bits < 32 && (1ll << bits) < cells) ++bits;
  tb = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, keys2, vals, id, n, 0, bits, s));
  CK(cub::DeviceRadixSort::SortPairs(ctx->tmp(tb), tb, keys, keys2, vals, id, n, 0, bits, s));
  LAUNCH(ctx);
  double* cols = dalloc<double>(gb.cols, 6 * (size_t)n);
  for (int a = 0; a < 6; ++a) g.x[a] = cols + (size_t)a * n;
  g.start = start;
  g.id = id;
  k_grid_gather<<<grid_for(n, 256), 256, 0, s>>>(S, id, g);
  LAUNCH(ctx);
  check_launch();
  g.ok = 1;
  return g;
}

// preprocess_object on the device: through the sample grid (cells of half
// the probe width) when it exists, else the all-pairs sweep.
void preprocess_device(lg_ctx* ctx, const DSamples& S, const DGrid& g, double h, double d,
                       uint8_t* keep, cudaStream_t s) {
  if (g.ok)
    k_preprocess_grid<<<grid_for(S.n, 128), 128, 0, s>>>(S, g, h, d, keep);
  else
    k_preprocess<<<grid_for(S.n, 256), 256, 0, s>>>(S, h, d, keep);
  LAUNCH(ctx);
  check_launch();
}

// place_object for candidates [c0, c0 + m) only (lg_place_batch): run_batch's
// stage-1 placement, then return the records.
struct PlaceOnly {
  int c0 = 0, m = 0;
  std::vector<double> pose, pen, stp, stn;
  std::vector<int> acc, nst, stl;
};

void run_batch_device(lg_ctx* ctx, const lg_hand_desc& hd, const lg_patches_desc& pd,
                      lg_field* field_in, const double* raw, int n_raw, const lg_run_params& cfg,
                      RunOut& out, PlaceOnly* place_only = nullptr) {
  auto wall0 = std::chrono::steady_clock::now();
  cudaStream_t s = ctx->stream;
  std::memset(&out.profile, 0, sizeof(out.profile));
  long long launches0 = ctx->launches;
  g_h2d = 0;
  g_d2h = 0;
  if (cfg.k_contacts < 1 || cfg.k_contacts > kMaxK) throw std::invalid_argument("k_contacts out of range");
  if (n_raw < 1) throw std::invalid_argument("place_object: no object samples");
  {
    unsigned long long z[kCntN] = {0, 0, 0, 0, 0};
    CK(cudaMemcpyToSymbolAsync(g_cnt, z, sizeof(z), 0, cudaMemcpyHostToDevice, s));
  }
  Timer tm(s);
  Timer tdev(s);   // device span of the pass after the inputs are resident
  Timer tk(s);     // per-kernel spans (realize, contact search)
  double realize_s = 0.0, copt_s = 0.0;
  // ---- field (ContactFieldIndex::build) or reuse
  // build_field (pipeline.cpp:286-304): with cfg.cache the index is read
  // from <out>/index_cache.bin when its key matches, else built and saved.
  std::unique_ptr<lg_field> own;
  lg_field* field = field_in;
  if (!field) {
    own.reset(new lg_field);
    own->ctx = ctx;
    uint64_t key = 0;
    std::string cache_path = std::string(cfg.out) + "/index_cache.bin";
    if (cfg.cache) {
      if (lg_index_cache_key(&cfg, &key) != LG_OK) {
        char msg[512];
        lg_last_error(msg, sizeof(msg));
        throw std::invalid_argument(msg);
      }
      if (!load_field(ctx, hd, cache_path.c_str(), key, own.get())) {
        own.reset(new lg_field);
        own->ctx = ctx;
      }
    }
    if (!own->from_cache) {
      build_field_device(ctx, hd, pd, cfg.field_configs, cfg.box_width, cfg.seed, cfg.codebook_size,
                         own.get());
      out.profile.field_build = own->build_ms * 1e-3;
      if (cfg.cache) {
        std::filesystem::create_directories(cfg.out);
        save_field(own.get(), cache_path.c_str(), key);
      }
    }
    field = own.get();
  } else {
    bind_hand(ctx, hd);
  }
  out.profile.index_from_cache = field->from_cache ? 1 : 0;
  const DField& F = field->f;
  DevPatches cache_patches;
  if (field->from_cache) {
    if (F.P != pd.n_patches) throw std::invalid_argument("run_batch: cached index does not match the hand's patches");
    upload_patches(ctx, pd, cache_patches);
  }
  const DevPatches& DP = field->from_cache ? cache_patches : field->patches;
  out.profile.patches = F.P;
  out.profile.boxes = F.B;
  out.profile.index_codes = field->n_codes;
  out.profile.field_vectors = field->n_vectors;
  out.profile.object_samples = n_raw;

  // ---- object samples (raw SoA) and preprocess_object
  tm.start();
  // one upload of the [n][6] rows, columns split on the device
  Buf raw_rows, raw_cols;
  const double* d_rows = dupload(raw_rows, raw, 6 * (size_t)n_raw, s);
  double* d_rawc = dalloc<double>(raw_cols, 6 * (size_t)std::max(n_raw, 1));
  k_soa_gather<<<grid_for(n_raw, 256), 256, 0, s>>>(n_raw, d_rows, nullptr, d_rawc);
  LAUNCH(ctx);
  check_launch();
  DSamples RS;
  RS.n = n_raw;
  for (int a = 0; a < 6; ++a) RS.x[a] = d_rawc + (size_t)a * n_raw;
  // LG_TIMING=1: host-clock marks after stream syncs, printed at the end
  const bool timing = std::getenv("LG_TIMING") != nullptr;
  std::vector<std::pair<const char*, double>> marks;
  auto mark = [&](const char* name) {
    if (!timing) return;
    cudaStreamSynchronize(s);
    marks.push_back({name, std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count()});
  };
  mark("inputs_uploaded");
  tdev.start();
  Buf keepb;
  uint8_t* d_keep = dalloc<uint8_t>(keepb, (size_t)n_raw);
  if (cfg.probe_half_width <= 0.0 || cfg.probe_depth_threshold < 0.0)
    throw std::invalid_argument("preprocess_object: bad probe dimensions");
  // raw-sample grid: preprocess here, the collision sweeps later
  GridBufs rgrid_b;
  const DGrid RG = build_grid(ctx, RS, raw, n_raw, 0.5 * cfg.probe_half_width, rgrid_b, s);
  preprocess_device(ctx, RS, RG, cfg.probe_half_width, cfg.probe_depth_threshold, d_keep, s);
  auto keep = ddownload(d_keep, (size_t)n_raw, s);
  std::vector<int> kept;
  for (int i = 0; i < n_raw; ++i)
    if (keep[i]) kept.push_back(i);
  const int ns = (int)kept.size();
  if (ns == 0) throw std::runtime_error("run_batch: preprocessing stripped every object sample");
  out.profile.field_samples = ns;
  Buf kept_b, fs_cols;
  const int* d_kept = dupload(kept_b, kept.data(), kept.size(), s);
  double* d_fsc = dalloc<double>(fs_cols, 6 * (size_t)ns);
  k_soa_gather<<<grid_for(ns, 256), 256, 0, s>>>(ns, d_rows, d_kept, d_fsc);
  LAUNCH(ctx);
  check_launch();
  DSamples FS;
  FS.n = ns;
  for (int a = 0; a < 6; ++a) FS.x[a] = d_fsc + (size_t)a * ns;

  // ---- groups, statics (collect_static_surface)
  int G = 0;
  std::vector<int> gol = groups_of(hd, &G);
  if (G > LG_MAX_GROUPS) throw std::invalid_argument("device: too many dependency groups (max 32)");
  std::vector<int> gop(DP.P);
  for (int p = 0; p < DP.P; ++p) gop[p] = gol[DP.h_link[p]];
  Buf gopb;
  int* d_gop = dupload(gopb, gop.data(), gop.size(), s);
  std::vector<int> sp_part, sp_link, pt_idx, pt_link;
  for (int l = 0; l < hd.n_links; ++l) {
    if (gol[l] != -1) continue;
    for (int p = 0; p < hd.n_parts; ++p)
      if (hd.part_link[p] == l) {
        sp_part.push_back(p);
        sp_link.push_back(l);
      }
  }
  for (int p = 0; p < DP.P; ++p) {
    if (gop[p] != -1) continue;
    for (int i = DP.h_point_off[p]; i < DP.h_point_off[p + 1]; ++i) {
      pt_idx.push_back(i);
      pt_link.push_back(DP.h_link[p]);
    }
  }
  const int n_sp = (int)sp_part.size(), n_ss = (int)pt_idx.size();
  Buf b_spp, b_spl, b_pti, b_ptl, b_ssp, b_ssn, b_spose, b_ssl;
  int* d_spp = dupload(b_spp, sp_part.data(), sp_part.size(), s);
  int* d_spl = dupload(b_spl, sp_link.data(), sp_link.size(), s);
  int* d_pti = dupload(b_pti, pt_idx.data(), pt_idx.size(), s);
  int* d_ptl = dupload(b_ptl, pt_link.data(), pt_link.size(), s);
  double* d_ssp = dalloc<double>(b_ssp, 3 * (size_t)n_ss);
  double* d_ssn = dalloc<double>(b_ssn, 3 * (size_t)n_ss);
  double* d_spose = dalloc<double>(b_spose, 12 * (size_t)n_sp);
  int* d_ssl = d_ptl;
  k_statics<<<1, 256, 0, s>>>(n_ss, d_pti, d_ptl, DP.pts.as<double>(), DP.nrm.as<double>(), n_sp,
                              d_spl, d_ssp, d_ssn, d_spose);
  LAUNCH(ctx);
  check_launch();

  // ---- shard
  const int B = cfg.batch;
  int c_lo = 0, c_hi = B;
  if (cfg.shard_count > 1) {
    c_lo = (int)((long long)cfg.shard_rank * B / cfg.shard_count);
    c_hi = (int)((long long)(cfg.shard_rank + 1) * B / cfg.shard_count);
  }
  if (place_only) {
    c_lo = place_only->c0;
    c_hi = place_only->c0 + place_only->m;
  }
  const int Bl = c_hi - c_lo;
  const int k = cfg.k_contacts;
  out.profile.candidates = (long long)cfg.passes * Bl;
  mark("preprocess_statics");
  double t_pre = tm.stop();

  // ---- per-candidate placement state (pass 0, reused by later passes)
  Buf b_pose, b_acc, b_pen, b_nst, b_stl, b_stp, b_stn, b_mask, b_cnt, b_aabb;
  double* d_pose = dalloc<double>(b_pose, 12 * (size_t)std::max(Bl, 1));
  int* d_acc = dalloc<int>(b_acc, (size_t)std::max(Bl, 1));
  double* d_pen = dalloc<double>(b_pen, (size_t)std::max(Bl, 1));
  int* d_nst = dalloc<int>(b_nst, (size_t)std::max(Bl, 1));
  int* d_stl = dalloc<int>(b_stl, (size_t)std::max(Bl, 1));
  double* d_stp = dalloc<double>(b_stp, 3 * (size_t)std::max(Bl, 1));
  double* d_stn = dalloc<double>(b_stn, 3 * (size_t)std::max(Bl, 1));
  uint32_t* d_mask = dalloc<uint32_t>(b_mask, (size_t)std::max(Bl, 1) * ns);
  int* d_cnt = dalloc<int>(b_cnt, (size_t)std::max(Bl, 1) * std::max(G, 1));
  double* d_aabb = dalloc<double>(b_aabb, 6 * (size_t)std::max(Bl, 1));
  CK(cudaMemsetAsync(d_stp, 0, 3 * sizeof(double) * std::max(Bl, 1), s));
  CK(cudaMemsetAsync(d_stn, 0, 3 * sizeof(double) * std::max(Bl, 1), s));

  std::vector<lg_trace> pass_tr;
  std::vector<double> h_pose;
  std::vector<int> h_acc, h_nst, h_stl, h_cnt;
  std::vector<double> h_pen, h_stp, h_stn;

  const int R = cfg.restarts;
  const long long per_restart = k + 2ll * cfg.n_outer * k * cfg.n_inner;
  const long long per_cand = (long long)R * per_restart;
  IkCfg ikc;
  ikc.beta = cfg.beta;
  ikc.step_clamp = cfg.step_clamp;
  ikc.residual_tol = cfg.residual_tol;
  ikc.damping_scale = cfg.damping_scale;
  ikc.damping_min = 1e-6;     // IkParams default (ik.hpp:27), not set by run_batch
  ikc.iterations = cfg.ik_iterations;
  ikc.max_backtracks = 10;    // IkParams default (ik.hpp:28)
  WOpts wo;
  wo.iterations = cfg.pgd_iterations;
  wo.warm_iterations = cfg.pgd_warm_iterations;
  wo.step = cfg.pgd_step;
  wo.max_bt = 20;
  CollCfg cc;
  cc.margin = cfg.penetration_margin;
  cc.raw = RS;
  cc.part_link = ctx->h_part_link.as<int>();
  cc.grid = RG;

  mark("candidate_state");
  for (int pass = 0; pass < cfg.passes && Bl > 0; ++pass) {
    // -------- stage 1: placement + domains (pass 0) + group pick
    tm.start();
    if (pass == 0) {
      PlaceCfg pc;
      pc.seed = cfg.seed;
      pc.c_lo = c_lo;
      pc.Bl = Bl;
      pc.mode = cfg.placement_mode;
      pc.static_prob = cfg.static_contact_prob;
      pc.margin = cfg.penetration_margin;
      for (int a = 0; a < 3; ++a) {
        pc.center[a] = cfg.canonical_center[a];
        pc.half[a] = cfg.canonical_half_extents[a];
      }
      pc.n_ss = n_ss;
      pc.ss_p = d_ssp;
      pc.ss_n = d_ssn;
      pc.ss_link = d_ssl;
      pc.P = DP.P;
      pc.patch_link = DP.link.as<int>();
      pc.point_off = DP.point_off.as<int>();
      pc.fp_off = DP.fp_off.as<int>();
      pc.fps = DP.fps.as<int>();
      pc.pts = DP.pts.as<double>();
      pc.nrm = DP.nrm.as<double>();
      k_place_pose<<<grid_for(Bl, 64), 64, 0, s>>>(pc, FS, d_pose, d_nst, d_stl, d_stp, d_stn);
      LAUNCH(ctx);
      check_launch();
      k_place_verdict<<<Bl, 256, 0, s>>>(Bl, FS, d_pose, n_sp, d_spp, d_spose, cfg.penetration_margin,
                                         d_acc, d_pen);
      LAUNCH(ctx);
      check_launch();
      if (place_only) {
        place_only->pose = ddownload(d_pose, 12 * (size_t)Bl, s);
        place_only->acc = ddownload(d_acc, (size_t)Bl, s);
        place_only->pen = ddownload(d_pen, (size_t)Bl, s);
        place_only->nst = ddownload(d_nst, (size_t)Bl, s);
        place_only->stl = ddownload(d_stl, (size_t)Bl, s);
        place_only->stp = ddownload(d_stp, 3 * (size_t)Bl, s);
        place_only->stn = ddownload(d_stn, 3 * (size_t)Bl, s);
        return;
      }
      if (ensure_dirlists(field, cfg.theta_hit)) {
        size_t qsm = codebook_smem(k_query3, F.C);
        k_query3<<<Bl, 256, qsm, s>>>(Bl, field->f, FS, d_pose, d_acc, cfg.theta_hit, G, qsm > 0,
                                      d_mask, d_cnt);
      } else if (F.grid_ok) {
        size_t qsm = codebook_smem(k_query2, F.C);
        k_query2<<<Bl, 256, qsm, s>>>(Bl, F, FS, d_pose, d_acc, cfg.theta_hit, G, qsm > 0, d_mask,
                                      d_cnt);
      } else {
        size_t qsm = codebook_smem(k_query, F.C);
        k_query<<<Bl, 256, qsm, s>>>(Bl, F, d_gop, FS, d_pose, d_acc, cfg.theta_hit, G, qsm > 0,
                                     d_mask, d_cnt);
      }
      LAUNCH(ctx);
      check_launch();
      k_obj_aabb<<<Bl, 256, 0, s>>>(Bl, RS, d_pose, d_acc, d_aabb);
      LAUNCH(ctx);
      check_launch();
    }
    Buf b_alive, b_chosen;
    int* d_alive = dalloc<int>(b_alive, (size_t)Bl);
    int* d_chosen = dalloc<int>(b_chosen, (size_t)Bl * kMaxK);
    k_group_pick<<<grid_for(Bl, 128), 128, 0, s>>>(Bl, c_lo, B, pass, cfg.seed, k, G, d_acc, d_cnt,
                                                    d_alive, d_chosen);
    LAUNCH(ctx);
    check_launch();
    auto h_alive = ddownload(d_alive, (size_t)Bl, s);
    auto h_chosen = ddownload(d_chosen, (size_t)Bl * kMaxK, s);
    if (pass == 0 || cfg.want_trace) {
      h_cnt = ddownload(d_cnt, (size_t)Bl * std::max(G, 1), s);
    }
    std::vector<int> alive_idx;
    for (int i = 0; i < Bl; ++i)
      if (h_alive[i]) alive_idx.push_back(i);
    const int nA = (int)alive_idx.size();
    out.profile.placements_accepted += nA;
    out.profile.placement_domains += tm.stop();

    if (cfg.want_trace) {
      if (pass == 0) {
        h_pose = ddownload(d_pose, 12 * (size_t)Bl, s);
        h_acc = ddownload(d_acc, (size_t)Bl, s);
        h_pen = ddownload(d_pen, (size_t)Bl, s);
        h_nst = ddownload(d_nst, (size_t)Bl, s);
        h_stl = ddownload(d_stl, (size_t)Bl, s);
        h_stp = ddownload(d_stp, 3 * (size_t)Bl, s);
        h_stn = ddownload(d_stn, 3 * (size_t)Bl, s);
      }
      pass_tr.assign(Bl, lg_trace());
      for (int i = 0; i < Bl; ++i) {
        lg_trace& t = pass_tr[i];
        std::memset(&t, 0, sizeof(t));
        t.g = (long long)pass * B + c_lo + i;
        t.pass = pass;
        t.c = c_lo + i;
        t.accepted = h_acc[i];
        t.penetration = h_pen[i];
        std::memcpy(t.pose_R, &h_pose[12 * i], 9 * sizeof(double));
        std::memcpy(t.pose_t, &h_pose[12 * i + 9], 3 * sizeof(double));
        t.n_static = h_nst[i];
        t.static_link = h_stl[i];
        if (h_nst[i]) {
          std::memcpy(t.static_p, &h_stp[3 * i], 3 * sizeof(double));
          std::memcpy(t.static_n, &h_stn[3 * i], 3 * sizeof(double));
        }
        t.n_groups = G;
        if (h_acc[i])
          for (int g = 0; g < G; ++g) t.domain_size[g] = h_cnt[(size_t)i * G + g];
        t.picked = h_alive[i];
        if (h_alive[i])
          for (int q = 0; q < k; ++q) t.chosen[q] = h_chosen[(size_t)i * kMaxK + q];
      }
    }
    if (nA == 0) {
      if (cfg.want_trace) out.traces.insert(out.traces.end(), pass_tr.begin(), pass_tr.end());
      continue;
    }

    mark("stage1");
    // -------- stage 2: contact optimisation
    tm.start();
    Buf b_aidx, b_eloff, b_els, b_elp, b_eln;
    int* d_aidx = dupload(b_aidx, alive_idx.data(), alive_idx.size(), s);
    std::vector<long long> eloff((size_t)nA * k + 1, 0);
    for (int a = 0; a < nA; ++a)
      for (int q = 0; q < k; ++q) {
        int i = alive_idx[a];
        eloff[(size_t)a * k + q + 1] =
            eloff[(size_t)a * k + q] + h_cnt[(size_t)i * G + h_chosen[(size_t)i * kMaxK + q]];
      }
    const long long nel = eloff.back();
    long long* d_eloff = dupload(b_eloff, eloff.data(), eloff.size(), s);
    // Large domains take the cooperative search over Morton-ordered copies
    // (dev_copt.cuh DomIdx; LG_PROJ=brute keeps the plain scan) and keep
    // only their sample ids: positions and normals are recomputed from the
    // sample and the pose where needed (ElemSrc), which saves writing and
    // re-reading 48 bytes per element.
    static const bool proj_brute = [] {
      const char* e = std::getenv("LG_PROJ");
      return e && std::string(e) == "brute";
    }();
    long long max_dom = 0;
    for (size_t t = 0; t + 1 < eloff.size(); ++t) max_dom = std::max(max_dom, eloff[t + 1] - eloff[t]);
    const bool large = !proj_brute && max_dom >= kCoopMin;
    int* d_els = dalloc<int>(b_els, (size_t)nel);
    // in a large run only the domains below kCoopMin (plain scan) are
    // materialised (the arrays keep the element indexing; the big domains'
    // ranges stay unwritten)
    const long long big_min = large ? kCoopMin : LLONG_MAX;
    double* d_elp = dalloc<double>(b_elp, 3 * (size_t)nel);
    double* d_eln = dalloc<double>(b_eln, 3 * (size_t)nel);
    k_domain_fill<<<(nA * k + 3) / 4, 128, 0, s>>>(nA, k, d_aidx, d_chosen, d_mask, FS, d_pose, d_eloff,
                                                   d_els, d_elp, d_eln, big_min);
    LAUNCH(ctx);
    check_launch();
    ElemSrc els{d_elp, d_eln, d_els, FS, d_pose, d_aidx, big_min};
    Buf b_keys, b_keys2, b_vals, b_vals2, b_sp, b_cb, b_sb, b_choff, b_suoff, b_cs, b_nch;
    DomIdx dom{};
    if (large) {
      const int nseg = nA * k;
      uint32_t* d_k = dalloc<uint32_t>(b_keys, (size_t)nel);
      uint32_t* d_k2 = dalloc<uint32_t>(b_keys2, (size_t)nel);
      int* d_v = dalloc<int>(b_vals, (size_t)nel);
      int* d_v2 = dalloc<int>(b_vals2, (size_t)nel);
      k_dom_keys<<<nseg, 256, 0, s>>>(nA, k, d_aidx, d_aabb, d_eloff, els, d_k, d_v);
      LAUNCH(ctx);
      check_launch();
      size_t tb = 0;
      CK(cub::DeviceSegmentedSort::SortPairs(nullptr, tb, d_k, d_k2, d_v, d_v2, (int)nel, nseg,
                                             d_eloff, d_eloff + 1, s));
      CK(cub::DeviceSegmentedSort::SortPairs(ctx->tmp(tb), tb, d_k, d_k2, d_v, d_v2, (int)nel, nseg,
                                             d_eloff, d_eloff + 1, s));
      LAUNCH(ctx);
      // chunk counts (runs of the Morton order split at jumps), then offsets
      int* d_nch = dalloc<int>(b_nch, (size_t)nseg);
      k_dom_chunk_count<<<nseg, 256, 0, s>>>(nseg, d_eloff, d_k2, d_nch);
      LAUNCH(ctx);
      check_launch();
      const std::vector<int> nch = ddownload(d_nch, (size_t)nseg, s);
      std::vector<long long> choff((size_t)nseg + 1, 0), suoff((size_t)nseg + 1, 0);
      for (int t = 0; t < nseg; ++t) {
        choff[t + 1] = choff[t] + nch[t];
        suoff[t + 1] = suoff[t] + (nch[t] + 31) / 32;
      }
      long long* d_choff = dupload(b_choff, choff.data(), choff.size(), s);
      long long* d_suoff = dupload(b_suoff, suoff.data(), suoff.size(), s);
      double* d_sp = dalloc<double>(b_sp, 3 * (size_t)nel);
      const long long cs = std::max(choff.back(), 1ll), ss = std::max(suoff.back(), 1ll);
      double* d_cb = dalloc<double>(b_cb, 6 * (size_t)cs);
      double* d_sb = dalloc<double>(b_sb, 6 * (size_t)ss);
      int* d_cs = dalloc<int>(b_cs, (size_t)cs);
      dom.sx = d_sp;
      dom.sy = d_sp + nel;
      dom.sz = d_sp + 2 * nel;
      dom.si = reinterpret_cast<int*>(d_k);  // the key buffer is free after the sort
      dom.cs = d_cs;
      dom.cb = d_cb;
      dom.cstride = cs;
      dom.sb = d_sb;
      dom.sstride = ss;
      dom.choff = d_choff;
      dom.suoff = d_suoff;
      k_dom_chunks<<<nseg, 256, 0, s>>>(nseg, d_eloff, d_choff, d_suoff, d_k2, d_v2, els, k, dom);
      LAUNCH(ctx);
      check_launch();
    }
    Buf b_draws, b_oid, b_oobj, b_oan, b_osol, b_bal;
    uint64_t* d_draws = dalloc<uint64_t>(b_draws, (size_t)nA * per_cand);
    {
      const int prp = cfg.n_outer * k * cfg.n_inner;  // Box-Muller pairs per restart
      k_copt_draws_warp<<<(nA + kDrawWarps - 1) / kDrawWarps, 32 * kDrawWarps, 0, s>>>(
          nA, d_aidx, c_lo, B, pass, cfg.seed, per_cand, per_restart, k, prp, cfg.sigma, d_draws);
      LAUNCH(ctx);
      check_launch();
    }
    int* d_oid = dalloc<int>(b_oid, (size_t)nA * kMaxK);
    double* d_oobj = dalloc<double>(b_oobj, (size_t)nA);
    int* d_oan = dalloc<int>(b_oan, (size_t)nA);
    double* d_osol = dalloc<double>(b_osol, (size_t)nA * 3 * kMaxC);
    int* d_bal = dalloc<int>(b_bal, (size_t)nA);
    CoptCfg co;
    co.k = k;
    co.n_outer = cfg.n_outer;
    co.n_inner = cfg.n_inner;
    co.restarts = R;
    co.sigma = cfg.sigma;
    co.lambda = cfg.lambda_torque;
    co.mu = cfg.mu;
    co.o = wo;
    co.per_restart = per_restart;
    co.per_cand = per_cand;
    int nw = std::min(R, 4);
    static const int co_minb = [] {
      const char* e = std::getenv("LG_COPT_MINB");
      return (e && std::atoi(e) == 5) ? 5 : 4;
    }();
    if (first_on_device(2)) {
      for (auto kern : {k_contact_opt2<3, 4, false>, k_contact_opt2<3, 5, false>,
                        k_contact_opt2<4, 4, false>, k_contact_opt2<kMaxC, 4, false>,
                        k_contact_opt2<3, 4, true>, k_contact_opt2<4, 4, true>,
                        k_contact_opt2<kMaxC, 4, true>})
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      // shared-memory carve-out (percent): less shared memory leaves more L1
      // for the domain scans, at the cost of resident CTAs
      const char* cv = std::getenv("LG_COPT_CARVE");
      if (cv) {
        int pct = std::atoi(cv);
        CK(cudaFuncSetAttribute(k_contact_opt2<3, 4, false>, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
        CK(cudaFuncSetAttribute(k_contact_opt2<3, 5, false>, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
      }
    }
    tk.start();
    // k contacts + at most one static
    // (the per-lane shared records scale with NC: NC = 4 fits three CTAs per
    // SM where NC = 6 fits two)
    const bool lg = dom.sx != nullptr;
    auto co_kern = k + 1 <= 3
                       ? (lg ? k_contact_opt2<3, 4, true>
                             : (co_minb == 5 ? k_contact_opt2<3, 5, false> : k_contact_opt2<3, 4, false>))
                   : k + 1 <= 4 ? (lg ? k_contact_opt2<4, 4, true> : k_contact_opt2<4, 4, false>)
                                : (lg ? k_contact_opt2<kMaxC, 4, true> : k_contact_opt2<kMaxC, 4, false>);
    size_t co_smem = k + 1 <= 3   ? copt2_smem<3>(k, nw)
                     : k + 1 <= 4 ? copt2_smem<4>(k, nw)
                                  : copt2_smem<kMaxC>(k, nw);
    co_kern<<<nA, 32 * nw, co_smem, s>>>(nA, d_aidx, co, d_nst, d_stp, d_stn, d_eloff, els, dom,
                                         d_draws, d_oid, d_oobj, d_oan, d_osol, cfg.eps_stable,
                                         d_bal);
    LAUNCH(ctx);
    check_launch();
    copt_s += tk.stop();
    auto h_bal = ddownload(d_bal, (size_t)nA, s);
    std::vector<int> bal_list;
    for (int a = 0; a < nA; ++a)
      if (h_bal[a]) bal_list.push_back(a);
    out.profile.contact_sets_balanced += (long long)bal_list.size();
    out.profile.contact_optimization += tm.stop();
    if (cfg.want_trace) {
      auto h_oid = ddownload(d_oid, (size_t)nA * kMaxK, s);
      auto h_oobj = ddownload(d_oobj, (size_t)nA, s);
      auto h_oan = ddownload(d_oan, (size_t)nA, s);
      auto h_osol = ddownload(d_osol, (size_t)nA * 3 * kMaxC, s);
      auto h_els = ddownload(d_els, (size_t)nel, s);
      for (int a = 0; a < nA; ++a) {
        lg_trace& t = pass_tr[alive_idx[a]];
        for (int q = 0; q < k; ++q) {
          t.opt_element[q] = h_oid[(size_t)a * kMaxK + q];
          t.opt_sample[q] = h_els[eloff[(size_t)a * k + q] + t.opt_element[q]];
        }
        t.opt_objective = h_oobj[a];
        t.opt_anchor = h_oan[a];
        t.opt_evaluations = R * (1 + cfg.n_outer * k * cfg.n_inner);
        int nc = k + h_nst[alive_idx[a]];
        for (int c = 0; c < nc; ++c) {
          t.opt_alpha[c] = h_osol[(size_t)a * 3 * kMaxC + c];
          t.opt_bx[c] = h_osol[(size_t)a * 3 * kMaxC + kMaxC + c];
          t.opt_by[c] = h_osol[(size_t)a * 3 * kMaxC + 2 * kMaxC + c];
        }
        t.balanced = h_bal[a];
      }
    }

    mark("stage2");
    // -------- stage 3: lookup attempts (reverse lookup + realize + filter)
    tm.start();
    Buf b_have, b_bclear, b_bres, b_bq, b_bused, b_btgt, b_blink, b_batt, b_runs;
    int* d_have = dalloc<int>(b_have, (size_t)nA);
    int* d_bclear = dalloc<int>(b_bclear, (size_t)nA);
    double* d_bres = dalloc<double>(b_bres, (size_t)nA);
    double* d_bq = dalloc<double>(b_bq, (size_t)nA * kMaxDof);
    auto* d_bused = dalloc<unsigned long long>(b_bused, (size_t)nA);
    double* d_btgt = dalloc<double>(b_btgt, (size_t)nA * kMaxK * 12);
    int* d_blink = dalloc<int>(b_blink, (size_t)nA * kMaxK);
    int* d_batt = dalloc<int>(b_batt, (size_t)nA);
    CK(cudaMemsetAsync(d_have, 0, sizeof(int) * nA, s));
    CK(cudaMemsetAsync(d_bclear, 0, sizeof(int) * nA, s));
    CK(cudaMemsetAsync(d_bq, 0, sizeof(double) * nA * kMaxDof, s));
    CK(cudaMemsetAsync(d_batt, 0xff, sizeof(int) * nA, s));
    Buf b_bal_l, b_tgt, b_tl, b_qt, b_res, b_fin, b_used, b_clean, b_on, b_cand, b_err, b_runs_d;
    int* d_err = dalloc<int>(b_err, 1);
    CK(cudaMemsetAsync(d_err, 0, sizeof(int), s));
    int* d_runs = dalloc<int>(b_runs_d, (size_t)nA);
    CK(cudaMemsetAsync(d_runs, 0, sizeof(int) * nA, s));
    const int nB = (int)bal_list.size();
    const int LA = cfg.lookup_attempts;
    const long long nP = (long long)nB * LA;  // every (candidate, attempt) problem
    if (nB > 0) {
      int* d_bl = dupload(b_bal_l, bal_list.data(), bal_list.size(), s);
      double* d_tgt = dalloc<double>(b_tgt, (size_t)nP * k * 12);
      int* d_tl = dalloc<int>(b_tl, (size_t)nP * k);
      k_targets_all<<<grid_for(nP * k, 128), 128, 0, s>>>(
          nB, d_bl, d_aidx, k, LA, c_lo, B, pass, cfg.seed, F, d_gop, DP.pts.as<double>(),
          DP.nrm.as<double>(), DP.link.as<int>(), d_chosen, d_oid, d_eloff, els,
          cfg.theta_hit, d_tgt, d_tl, d_err);
      LAUNCH(ctx);
      check_launch();
      double* d_qt = dalloc<double>(b_qt, (size_t)nP * kMaxDof);
      double* d_res = dalloc<double>(b_res, (size_t)nP);
      int* d_fin = dalloc<int>(b_fin, (size_t)nP);
      auto* d_used = dalloc<unsigned long long>(b_used, (size_t)nP);
      tk.start();
      launch_realize_warp(s, (int)nP, k, nullptr, ikc, cfg.finetune_rounds, cfg.finetune_iterations,
                          d_tgt, k * 12, d_tl, k, nullptr, d_qt, d_res, d_fin, d_used, hd.dof,
                          hd.n_links);
      LAUNCH(ctx);
      check_launch();
      realize_s += tk.stop();
      out.profile.realize_calls += nP;
      int* d_on = dalloc<int>(b_on, (size_t)nP);
      k_conv_flags<<<grid_for(nP, 256), 256, 0, s>>>((int)nP, d_fin, d_res, cfg.contact_tol, d_on);
      LAUNCH(ctx);
      std::vector<int> cand(nP);
      for (long long p = 0; p < nP; ++p) cand[p] = alive_idx[bal_list[p / LA]];
      int* d_cand = dupload(b_cand, cand.data(), cand.size(), s);
      uint8_t* d_clean = dalloc<uint8_t>(b_clean, (size_t)nP);
      CK(cudaMemsetAsync(d_clean, 0, nP, s));
      coll_kernel(cc)<<<((int)nP + kCollWarps - 1) / kCollWarps, 32 * kCollWarps, 0, s>>>(
          (int)nP, cc, d_cand, d_on, d_qt, d_pose, d_aabb, 1,
                                            d_clean, nullptr);
      LAUNCH(ctx);
      check_launch();
      k_attempt_select<<<grid_for(nB, 128), 128, 0, s>>>(
          nB, d_bl, k, LA, d_qt, d_res, d_fin, d_used, d_clean, d_tgt, d_tl, cfg.contact_tol, d_have,
          d_bclear, d_bres, d_bq, d_bused, d_btgt, d_blink, d_batt, d_runs);
      LAUNCH(ctx);
      check_launch();
      auto h_on = ddownload(d_on, (size_t)nP, s);
      for (long long p = 0; p < nP; ++p) out.profile.collision_calls += h_on[p];
    }
    std::vector<int> attempts_run = ddownload(d_runs, (size_t)nA, s);
    int herr = 0;
    CK(cudaMemcpyAsync(&herr, d_err, sizeof(int), cudaMemcpyDeviceToHost, s));
    auto h_have = ddownload(d_have, (size_t)nA, s);
    if (herr) throw std::out_of_range("reverse_lookup: element has no hits");
    std::vector<int> real_list;
    for (int a = 0; a < nA; ++a)
      if (h_have[a]) real_list.push_back(a);
    out.profile.ik_finite += (long long)real_list.size();
    out.profile.kinematics_optimization += tm.stop();
    if (cfg.want_trace) {
      auto h_bclear = ddownload(d_bclear, (size_t)nA, s);
      auto h_bres = ddownload(d_bres, (size_t)nA, s);
      auto h_bq = ddownload(d_bq, (size_t)nA * kMaxDof, s);
      auto h_bused = ddownload(d_bused, (size_t)nA, s);
      auto h_btgt = ddownload(d_btgt, (size_t)nA * kMaxK * 12, s);
      auto h_blink = ddownload(d_blink, (size_t)nA * kMaxK, s);
      auto h_batt = ddownload(d_batt, (size_t)nA, s);
      for (int a = 0; a < nA; ++a) {
        if (!h_bal[a]) continue;
        lg_trace& t = pass_tr[alive_idx[a]];
        t.realized = h_have[a];
        t.attempts_run = attempts_run[a];
        t.best_attempt = h_have[a] ? h_batt[a] : -1;
        t.best_clear = h_bclear[a];
        if (h_have[a]) {
          t.max_residual = h_bres[a];
          for (int j = 0; j < hd.dof; ++j) t.real_q[j] = h_bq[(size_t)a * kMaxDof + j];
          t.used_joints = h_bused[a];
          for (int q = 0; q < k; ++q) {
            t.target_link[q] = h_blink[(size_t)a * kMaxK + q];
            std::memcpy(t.target_point[q], &h_btgt[((size_t)a * kMaxK + q) * 12 + 6], 3 * sizeof(double));
            std::memcpy(t.target_normal[q], &h_btgt[((size_t)a * kMaxK + q) * 12 + 9], 3 * sizeof(double));
          }
        }
      }
    }
    if (real_list.empty()) {
      if (cfg.want_trace) out.traces.insert(out.traces.end(), pass_tr.begin(), pass_tr.end());
      continue;
    }

    mark("stage3");
    // -------- stage 4: unused-joint redraws + postprocess
    tm.start();
    Buf b_fq, b_fclean, b_uatt, b_grasp, b_valid, b_drop, b_act_r, b_qall;
    double* d_fq = dalloc<double>(b_fq, (size_t)nA * kMaxDof);
    uint8_t* d_fclean = dalloc<uint8_t>(b_fclean, (size_t)nA);
    const int nR = (int)real_list.size();
    const int UA = cfg.unused_attempts;
    const long long nU = (long long)nR * UA;  // every (candidate, redraw) configuration
    int* d_real = dupload(b_act_r, real_list.data(), real_list.size(), s);
    double* d_qall = dalloc<double>(b_qall, (size_t)nU * kMaxDof);
    k_unused_all<<<grid_for(nR, 64), 64, 0, s>>>(nR, d_real, d_aidx, UA, c_lo, B, pass, cfg.seed, d_bq,
                                                 d_bused, d_qall);
    LAUNCH(ctx);
    check_launch();
    mark("post_unused_draws");
    {
      std::vector<int> cand(nU);
      for (long long u = 0; u < nU; ++u) cand[u] = alive_idx[real_list[u / UA]];
      int* d_cand = dupload(b_cand, cand.data(), cand.size(), s);
      uint8_t* d_clean = dalloc<uint8_t>(b_clean, (size_t)nU);
      out.profile.collision_calls += nU;
      coll_kernel(cc)<<<((int)nU + kCollWarps - 1) / kCollWarps, 32 * kCollWarps, 0, s>>>(
          (int)nU, cc, d_cand, nullptr, d_qall, d_pose, d_aabb, 1,
                                            d_clean, nullptr);
      LAUNCH(ctx);
      check_launch();
      int* d_uatt_d = dalloc<int>(b_uatt, (size_t)nA);
      CK(cudaMemsetAsync(d_uatt_d, 0xff, sizeof(int) * nA, s));
      CK(cudaMemsetAsync(d_fclean, 0, nA, s));
      k_unused_select<<<grid_for(nR, 128), 128, 0, s>>>(nR, d_real, UA, d_qall, d_clean, d_fq, d_fclean,
                                                        d_uatt_d);
      LAUNCH(ctx);
      check_launch();
    }
    lg_grasp* d_grasp = dalloc<lg_grasp>(b_grasp, (size_t)nA);
    int* d_valid = dalloc<int>(b_valid, (size_t)nA);
    int* d_drop = dalloc<int>(b_drop, (size_t)nA);
    CK(cudaMemsetAsync(d_grasp, 0, sizeof(lg_grasp) * nA, s));
    CK(cudaMemsetAsync(d_valid, 0, sizeof(int) * nA, s));
    CK(cudaMemsetAsync(d_drop, 0, sizeof(int) * nA, s));
    FinalCfg fc;
    fc.k = k;
    fc.contact_tol = cfg.contact_tol;
    fc.lambda = cfg.lambda_torque;
    fc.mu = cfg.mu;
    fc.eps = cfg.eps_stable;
    fc.o = wo;
    k_finalize_warp<<<(nR + 3) / 4, 128, 0, s>>>(nR, d_real, d_aidx, fc, FS, d_pose, d_nst, d_stl, d_stp,
                                                 d_stn, d_fq, d_fclean, d_btgt, d_blink, d_grasp,
                                                 d_valid, d_drop);
    LAUNCH(ctx);
    check_launch();
    mark("post_finalize");
    std::vector<int> uatt;
    std::vector<double> fq_h;
    std::vector<lg_grasp> h_grasp;
    std::vector<int> h_valid, h_drop;
    if (cfg.want_trace) {
      uatt = ddownload(b_uatt.as<int>(), (size_t)nA, s);
      fq_h = ddownload(d_fq, (size_t)nA * kMaxDof, s);
      h_grasp = ddownload(d_grasp, (size_t)nA, s);
      h_valid = ddownload(d_valid, (size_t)nA, s);
      h_drop = ddownload(d_drop, (size_t)nA, s);
      for (int a : real_list) {
        const lg_grasp& g = h_grasp[a];
        if (!h_drop[a]) {
          out.profile.penetration_free += g.penetration_free;
          out.profile.ik_converged += g.ik_converged;
          out.profile.stable += g.stable;
        }
      }
      // kept grasps in candidate order (pipeline.cpp:607-614)
      for (int a = 0; a < nA; ++a) {
        if (!h_valid[a] || h_drop[a]) continue;
        lg_grasp g = h_grasp[a];
        g.g = (long long)pass * B + c_lo + alive_idx[a];
        out.grasps.push_back(g);
      }
    } else {
      // funnel counts and the kept grasps compacted on the device (stable
      // selection keeps candidate order): only the kept records cross PCIe
      Buf b_keep, b_sel, b_nsel, b_fl;
      uint8_t* d_keep8 = dalloc<uint8_t>(b_keep, (size_t)nA);
      int* d_fl = dalloc<int>(b_fl, 3);
      CK(cudaMemsetAsync(d_fl, 0, 3 * sizeof(int), s));
      k_grasp_flags<<<grid_for(nA, 256), 256, 0, s>>>(nA, d_grasp, d_valid, d_drop, d_keep8, d_fl);
      LAUNCH(ctx);
      check_launch();
      lg_grasp* d_sel = dalloc<lg_grasp>(b_sel, (size_t)nA);
      int* d_nsel = dalloc<int>(b_nsel, 1);
      Buf b_dest;
      int* d_dest = dalloc<int>(b_dest, (size_t)nA);
      k_compact_rank<<<1, 1024, 0, s>>>(nA, d_keep8, d_dest, d_nsel);
      LAUNCH(ctx);
      check_launch();
      k_copy_grasps<<<grid_for((long long)nA * 32, 256), 256, 0, s>>>(nA, d_grasp, d_dest, d_sel);
      LAUNCH(ctx);
      check_launch();
      int counts[4];
      CK(cudaMemcpyAsync(counts, d_fl, 3 * sizeof(int), cudaMemcpyDeviceToHost, s));
      CK(cudaMemcpyAsync(counts + 3, d_nsel, sizeof(int), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      g_d2h += 4 * sizeof(int);
      out.profile.penetration_free += counts[0];
      out.profile.ik_converged += counts[1];
      out.profile.stable += counts[2];
      auto sel = ddownload(d_sel, (size_t)counts[3], s);
      std::vector<int> kept_a;  // candidate index of each kept grasp, in order
      {
        auto keep8 = ddownload(d_keep8, (size_t)nA, s);
        for (int a = 0; a < nA; ++a)
          if (keep8[a]) kept_a.push_back(a);
      }
      for (size_t t = 0; t < sel.size(); ++t) {
        lg_grasp g = sel[t];
        g.g = (long long)pass * B + c_lo + alive_idx[kept_a[t]];
        out.grasps.push_back(g);
      }
    }
    out.profile.postprocessing += tm.stop();
    if (cfg.want_trace) {
      for (int a : real_list) {
        lg_trace& t = pass_tr[alive_idx[a]];
        t.unused_attempt = uatt[a];
        for (int j = 0; j < hd.dof; ++j) t.final_q[j] = fq_h[(size_t)a * kMaxDof + j];
        t.dropped = h_drop[a];
        if (!h_drop[a]) {
          t.penetration_free = h_grasp[a].penetration_free;
          t.ik_converged = h_grasp[a].ik_converged;
          t.stable = h_grasp[a].stable;
          t.valid = h_valid[a];
          t.objective = h_grasp[a].objective;
        }
      }
      out.traces.insert(out.traces.end(), pass_tr.begin(), pass_tr.end());
    }
  }
  mark("passes_done");
  if (timing)
    for (auto& m : marks) std::fprintf(stderr, "[lg timing] %-20s %9.3f ms\n", m.first, 1e3 * m.second);
    std::fprintf(stderr, "[lg timing] cudaMalloc calls so far %lld, %.3f ms\n", g_malloc_calls, g_malloc_ms);
  out.profile.valid = (long long)out.grasps.size();
  out.profile.device_seconds = tdev.stop() + out.profile.field_build;
  {
    unsigned long long c[kCntN];
    CK(cudaMemcpyFromSymbol(c, g_cnt, sizeof(c)));
    out.profile.ik_iterations = (long long)c[kCntIk];
    out.profile.fk_evals = (long long)c[kCntFk];
    out.profile.wrench_evals = (long long)c[kCntWeval];
    out.profile.wrench_grads = (long long)c[kCntWgrad];
    out.profile.proj_evals = (long long)c[kCntProj];
  }
  out.profile.realize_seconds = realize_s;
  out.profile.contact_opt_seconds = copt_s;
  out.profile.h2d_bytes = g_h2d;
  out.profile.d2h_bytes = g_d2h;
  double total = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
  (void)t_pre;
  out.profile.total = total;
  out.profile.grasps_per_second = total > 0.0 ? out.profile.valid / total : 0.0;
  out.profile.gpu_launches = ctx->launches - launches0;
}

}  // namespace

struct lg_result {
  RunOut r;
};

namespace {

// Stage-level batch kernels for the parity harness.
__global__ void k_wrench_batch(int m, const int* n, const double* pts, const double* nrm,
                               double lambda, double mu, int mode, WOpts o, double* obj,
                               int* anchor, double* sol) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  WProb w;
  w.n = n[t];
  w.lambda = lambda;
  w.mu = mode ? mu : 0.0;  // solve_gswo with mu == 0 is solve_fswo
  for (int c = 0; c < w.n; ++c)
    wprob_set(w, c, v3_load(pts + (size_t)t * 18 + 3 * c), v3_load(nrm + (size_t)t * 18 + 3 * c));
  WState s;
  int an = -1;
  Ctr ctr = {0, 0, 0, 0, 0};
  double v = wsolve(w, o, nullptr, &an, s, ctr);
  obj[t] = v;
  anchor[t] = an;
  for (int c = 0; c < kMaxC; ++c) {
    sol[(size_t)t * 18 + c] = s.a[c];
    sol[(size_t)t * 18 + 6 + c] = s.bx[c];
    sol[(size_t)t * 18 + 12 + c] = s.by[c];
  }
}

// Explicit WrenchProblems (caller tangents, per-problem lambda and mu) with
// optional warm starts: run_solver (wrench.cpp:179-228) per thread.
__global__ void k_wrench_problems(int m, const int* n, const double* pts, const double* nrm,
                                  const double* tx, const double* ty, const double* lambda,
                                  const double* mu, int mode, WOpts o, const int* use_warm,
                                  const double* warm, double* obj, int* anchor, double* sol) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  WProb w;
  w.n = n[t];
  w.lambda = lambda[t];
  w.mu = mode ? mu[t] : 0.0;
  for (int c = 0; c < w.n; ++c) {
    const size_t b = (size_t)t * 18 + 3 * c;
    const V3 p = v3_load(pts + b);
    w.p[c] = p;
    w.nn[c] = v3_load(nrm + b);
    w.tx[c] = v3_load(tx + b);
    w.ty[c] = v3_load(ty + b);
    w.cn[c] = cross(p, w.nn[c]);  // Precomp (wrench.cpp:50-64)
    w.cx[c] = cross(p, w.tx[c]);
    w.cy[c] = cross(p, w.ty[c]);
  }
  WState ws;
  const bool wm = use_warm && use_warm[t];
  if (wm)
    for (int c = 0; c < kMaxC; ++c) {
      ws.a[c] = warm[(size_t)t * 18 + c];
      ws.bx[c] = warm[(size_t)t * 18 + 6 + c];
      ws.by[c] = warm[(size_t)t * 18 + 12 + c];
    }
  WState s;
  int an = -1;
  Ctr ctr = {0, 0, 0, 0, 0};
  double v = wsolve(w, o, wm ? &ws : nullptr, &an, s, ctr);
  obj[t] = v;
  anchor[t] = an;
  for (int c = 0; c < kMaxC; ++c) {
    sol[(size_t)t * 18 + c] = s.a[c];
    sol[(size_t)t * 18 + 6 + c] = s.bx[c];
    sol[(size_t)t * 18 + 12 + c] = s.by[c];
  }
}

}  // namespace

extern "C" {

int lg_wrench_problem_batch(lg_ctx* ctx, int m, const int* n, const double* points,
                            const double* normals, const double* tangent_x,
                            const double* tangent_y, const double* lambda_torque,
                            const double* mu, int mode, int iterations, int warm_iterations,
                            double step, int max_backtracks, const int* use_warm,
                            const double* warm_alpha, const double* warm_beta_x,
                            const double* warm_beta_y, double* objective, int* anchor,
                            double* alpha, double* beta_x, double* beta_y) {
  return lgc::guard([&] {
    if (!ctx || m < 0 || (m > 0 && (!n || !points || !normals || !tangent_x || !tangent_y ||
                                    !lambda_torque || !mu || !objective || !anchor || !alpha ||
                                    !beta_x || !beta_y)))
      throw std::invalid_argument("lg_wrench_problem_batch: bad argument");
    for (int i = 0; i < m; ++i) {
      if (n[i] < 1) throw std::invalid_argument("wrench solve: no contacts");
      if (n[i] > kMaxC) throw std::invalid_argument("wrench solve: the device takes 1..6 contacts");
    }
    if (m == 0) return;
    use_ctx(ctx);
    cudaStream_t s = ctx->stream;
    std::vector<double> warm;
    if (use_warm) {
      if (!warm_alpha || !warm_beta_x || !warm_beta_y)
        throw std::invalid_argument("lg_wrench_problem_batch: warm arrays missing");
      warm.assign((size_t)m * 18, 0.0);
      for (int i = 0; i < m; ++i)
        for (int c = 0; c < kMaxC; ++c) {
          warm[(size_t)i * 18 + c] = warm_alpha[6 * i + c];
          warm[(size_t)i * 18 + 6 + c] = warm_beta_x[6 * i + c];
          warm[(size_t)i * 18 + 12 + c] = warm_beta_y[6 * i + c];
        }
    }
    Buf bn, bp, bq, bx, by, bl, bm, bu, bw, bo, ba, bs;
    int* d_n = dupload(bn, n, (size_t)m, s);
    double* d_p = dupload(bp, points, (size_t)m * 18, s);
    double* d_q = dupload(bq, normals, (size_t)m * 18, s);
    double* d_x = dupload(bx, tangent_x, (size_t)m * 18, s);
    double* d_y = dupload(by, tangent_y, (size_t)m * 18, s);
    double* d_l = dupload(bl, lambda_torque, (size_t)m, s);
    double* d_m = dupload(bm, mu, (size_t)m, s);
    int* d_u = use_warm ? dupload(bu, use_warm, (size_t)m, s) : nullptr;
    double* d_w = use_warm ? dupload(bw, warm.data(), warm.size(), s) : nullptr;
    double* d_o = dalloc<double>(bo, (size_t)m);
    int* d_a = dalloc<int>(ba, (size_t)m);
    double* d_s = dalloc<double>(bs, (size_t)m * 18);
    WOpts o;
    o.iterations = iterations;
    o.warm_iterations = warm_iterations;
    o.step = step;
    o.max_bt = max_backtracks;
    k_wrench_problems<<<grid_for(m, 64), 64, 0, s>>>(m, d_n, d_p, d_q, d_x, d_y, d_l, d_m, mode, o,
                                                     d_u, d_w, d_o, d_a, d_s);
    LAUNCH(ctx);
    check_launch();
    auto h_s = ddownload(d_s, (size_t)m * 18, s);
    auto h_o = ddownload(d_o, (size_t)m, s);
    auto h_a = ddownload(d_a, (size_t)m, s);
    for (int i = 0; i < m; ++i) {
      objective[i] = h_o[i];
      anchor[i] = h_a[i];
      for (int c = 0; c < kMaxC; ++c) {
        alpha[6 * i + c] = h_s[18 * i + c];
        beta_x[6 * i + c] = h_s[18 * i + 6 + c];
        beta_y[6 * i + c] = h_s[18 * i + 12 + c];
      }
    }
  });
}

int lg_wrench_solve_batch(lg_ctx* ctx, int m, const int* n, const double* points,
                          const double* normals, double lambda, double mu, int mode,
                          int iterations, int warm_iterations, double step, int max_backtracks,
                          double* objective, int* anchor, double* alpha, double* beta_x,
                          double* beta_y) {
  return lgc::guard([&] {
    if (!ctx || m < 0) throw std::invalid_argument("lg_wrench_solve_batch: bad argument");
    for (int i = 0; i < m; ++i)
      if (n[i] < 1 || n[i] > kMaxC) throw std::invalid_argument("wrench solve: 1..6 contacts");
    if (m == 0) return;
    use_ctx(ctx);
    cudaStream_t s = ctx->stream;
    Buf bn, bp, bq, bo, ba, bs;
    int* d_n = dupload(bn, n, (size_t)m, s);
    double* d_p = dupload(bp, points, (size_t)m * 18, s);
    double* d_q = dupload(bq, normals, (size_t)m * 18, s);
    double* d_o = dalloc<double>(bo, (size_t)m);
    int* d_a = dalloc<int>(ba, (size_t)m);
    double* d_s = dalloc<double>(bs, (size_t)m * 18);
    WOpts o;
    o.iterations = iterations;
    o.warm_iterations = warm_iterations;
    o.step = step;
    o.max_bt = max_backtracks;
    k_wrench_batch<<<grid_for(m, 64), 64, 0, s>>>(m, d_n, d_p, d_q, lambda, mu, mode, o, d_o, d_a, d_s);
    check_launch();
    auto h_s = ddownload(d_s, (size_t)m * 18, s);
    CK(cudaMemcpyAsync(objective, d_o, sizeof(double) * m, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(anchor, d_a, sizeof(int) * m, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (int i = 0; i < m; ++i)
      for (int c = 0; c < kMaxC; ++c) {
        alpha[6 * i + c] = h_s[18 * i + c];
        beta_x[6 * i + c] = h_s[18 * i + 6 + c];
        beta_y[6 * i + c] = h_s[18 * i + 12 + c];
      }
  });
}

// decompose_patches output (contact_field.hpp:20-30) owned by the library.
struct lg_patches {
  std::vector<int> link, point_off, fp_off, fps;
  std::vector<double> pts, nrm;
};

namespace {
// TriMesh face quantities (mesh.cpp:16-31) on one link's visual mesh.
struct VisMesh {
  const lg_visual_desc* d;
  int l;
  V3 vert(int t, int c) const {
    const int v = d->vert_off[l] + d->tris[3 * (d->tri_off[l] + t) + c];
    return v3_load(d->verts + 3 * v);
  }
  int ntri() const { return d->tri_off[l + 1] - d->tri_off[l]; }
  int nvert() const { return d->vert_off[l + 1] - d->vert_off[l]; }
  V3 face_normal(int t) const {
    V3 n = cross(sub(vert(t, 1), vert(t, 0)), sub(vert(t, 2), vert(t, 0)));
    double len = norm(n);
    if (len < 1e-300) return v3(0, 0, 1);
    return divs(n, len);
  }
  double face_area(int t) const {
    return 0.5 * norm(cross(sub(vert(t, 1), vert(t, 0)), sub(vert(t, 2), vert(t, 0))));
  }
  double surface_area() const {
    double a = 0.0;
    for (int t = 0; t < ntri(); ++t) a += face_area(t);
    return a;
  }
};
}  // namespace

int lg_patches_export(const lg_patches* p, lg_patches_desc* d) {
  return lgc::guard([&] {
    if (!p || !d) throw std::invalid_argument("lg_patches_export: null argument");
    d->n_patches = (int)p->link.size();
    d->link = p->link.data();
    d->point_off = p->point_off.data();
    d->points = p->pts.data();
    d->normals = p->nrm.data();
    d->fp_off = p->fp_off.data();
    d->field_points = p->fps.data();
  });
}
void lg_patches_destroy(lg_patches* p) { delete p; }

int lg_hand_patches_device(lg_ctx* ctx, const lg_hand_desc* hand, const lg_visual_desc* visual,
                           double spc, double radius, uint64_t seed, int cap, lg_patches** out) {
  return lgc::guard([&] {
    if (!ctx || !hand || !visual || !out)
      throw std::invalid_argument("lg_hand_patches_device: null argument");
    if (visual->n_links != hand->n_links)
      throw std::invalid_argument("decompose_patches: per-link sample mismatch");
    use_ctx(ctx);
    cudaStream_t s = ctx->stream;
    // per-link hand samples, stream 'hnds' (pipeline.cpp:277-285), on the
    // device: face areas / normals / counts on the host (O(triangles)), the
    // draws and points on the GPU (k_sample_draws, k_sample_points)
    std::vector<int> seg_link;
    std::vector<long long> off{0};
    std::vector<SampleSeg> segs;
    std::vector<double> corners, fn, cum;
    for (int l = 0; l < hand->n_links; ++l) {
      VisMesh m{visual, l};
      if (m.nvert() == 0 || m.ntri() == 0) continue;
      size_t count = (size_t)std::llround(m.surface_area() * 1e4 * spc);
      if (count == 0) count = 1;
      SampleSeg sg;
      sg.tri0 = (long long)cum.size();
      sg.s0 = off.back();
      sg.ntri = m.ntri();
      sg.count = (int)count;
      sg.seed = lgm::mix_seed(seed, 0x686e6473ull, (uint64_t)l);
      double acc = 0.0;
      for (int t = 0; t < m.ntri(); ++t) {
        acc += m.face_area(t);
        cum.push_back(acc);
        for (int c = 0; c < 3; ++c) {
          const V3 v = m.vert(t, c);
          corners.insert(corners.end(), {v.x, v.y, v.z});
        }
        V3 nn = m.face_normal(t);
        fn.insert(fn.end(), {nn.x, nn.y, nn.z});
      }
      segs.push_back(sg);
      seg_link.push_back(l);
      off.push_back(off.back() + (long long)count);
    }
    if (radius <= 0.0 || cap < 1) throw std::invalid_argument("decompose_patches: bad radius or cap");
    if (cap > 16) throw std::invalid_argument("lg_hand_patches_device: field cap above 16");
    const long long total = off.back();
    if (total == 0) throw std::invalid_argument("decompose_patches: no surface samples");
    const int nseg = (int)seg_link.size();
    Buf bsg, bss, bcr, bfn, bcu, bdr, bp, bnr;
    const SampleSeg* d_sg = dupload(bsg, segs.data(), segs.size(), s);
    const long long* d_ss = dupload(bss, off.data(), (size_t)nseg, s);
    const double* d_cr = dupload(bcr, corners.data(), corners.size(), s);
    const double* d_fn = dupload(bfn, fn.data(), fn.size(), s);
    const double* d_cu = dupload(bcu, cum.data(), cum.size(), s);
    uint64_t* d_dr = dalloc<uint64_t>(bdr, 3 * (size_t)total);
    double* d_p = dalloc<double>(bp, 3 * (size_t)total);
    double* d_nr = dalloc<double>(bnr, 3 * (size_t)total);
    k_sample_draws<<<grid_for(nseg, 32), 32, 0, s>>>(nseg, d_sg, d_dr);
    check_launch();
    k_sample_points<<<grid_for(total, 256), 256, 0, s>>>(total, nseg, d_sg, d_ss, d_cr, d_fn, d_cu, d_dr,
                                                          d_p, d_nr);
    check_launch();
    auto pos = ddownload(d_p, 3 * (size_t)total, s);
    auto nrm = ddownload(d_nr, 3 * (size_t)total, s);
    Buf bl, bo, ba, bb, bm, bs, bn;
    const int* d_l = dupload(bl, seg_link.data(), seg_link.size(), s);
    const long long* d_o = dupload(bo, off.data(), off.size(), s);
    int* d_a = dalloc<int>(ba, (size_t)total);
    int* d_b = dalloc<int>(bb, (size_t)total);
    int* d_m = dalloc<int>(bm, (size_t)total);
    int* d_s = dalloc<int>(bs, (size_t)total);
    int* d_n = dalloc<int>(bn, (size_t)nseg);
    k_patch_cover<<<nseg, kCoverThreads, 0, s>>>(nseg, d_l, d_o, d_p, 0.5 * radius, seed, d_a, d_b,
                                                 d_m, d_s, d_n);
    check_launch();
    auto members = ddownload(d_m, (size_t)total, s);
    auto pstart = ddownload(d_s, (size_t)total, s);
    auto npatch = ddownload(d_n, (size_t)nseg, s);
    // global patch order = link order, then cover order (patch.id)
    std::vector<int> msize, fp_off{0};
    auto* P = new lg_patches;
    std::unique_ptr<lg_patches> own(P);
    lg_patches& R = *P;
    R.point_off.push_back(0);
    R.fp_off.push_back(0);
    for (int b = 0; b < nseg; ++b) {
      const long long base = off[b];
      const int N = (int)(off[b + 1] - base);
      for (int k = 0; k < npatch[b]; ++k) {
        int st = pstart[base + k], en = k + 1 < npatch[b] ? pstart[base + k + 1] : N;
        R.link.push_back(seg_link[b]);
        for (int i = st; i < en; ++i) {
          long long g = base + members[base + i];
          R.pts.insert(R.pts.end(), {pos[3 * g], pos[3 * g + 1], pos[3 * g + 2]});
          R.nrm.insert(R.nrm.end(), {nrm[3 * g], nrm[3 * g + 1], nrm[3 * g + 2]});
        }
        R.point_off.push_back((int)(R.pts.size() / 3));
        msize.push_back(en - st);
        fp_off.push_back(fp_off.back() + std::min(en - st, cap));
      }
    }
    const int np = (int)msize.size();
    std::vector<int> gid(np);
    for (int t = 0; t < np; ++t) gid[t] = t;
    Buf bg, bz, bf, bq;
    const int* d_g = dupload(bg, gid.data(), gid.size(), s);
    const int* d_z = dupload(bz, msize.data(), msize.size(), s);
    const int* d_f = dupload(bf, fp_off.data(), fp_off.size(), s);
    int* d_q = dalloc<int>(bq, (size_t)fp_off.back());
    k_patch_fields<<<grid_for(np, 128), 128, 0, s>>>(np, d_g, d_z, d_f, cap, seed, d_q);
    check_launch();
    R.fps = ddownload(d_q, (size_t)fp_off.back(), s);
    R.fp_off = fp_off;
    *out = own.release();
  });
}

int lg_validate_batch(lg_ctx* ctx, const lg_hand_desc* hand, const lg_grasp* grasps, long long n,
                      const double* obj_verts, int nv, const int* obj_tris, int nt,
                      const double* samples, int ns, const lg_run_params* p,
                      lg_grasp_check* out) {
  return lgc::guard([&] {
    if (!ctx || !hand || !p || (n && (!grasps || !out)))
      throw std::invalid_argument("lg_validate_batch: null argument");
    if (nv < 0 || nt < 0 || ns < 0 || (nt && (!obj_verts || !obj_tris)) || (ns && !samples))
      throw std::invalid_argument("lg_validate_batch: bad object arrays");
    if (n == 0) return;
    use_ctx(ctx);
    cudaStream_t s = ctx->stream;
    bind_hand(ctx, *hand);
    for (int t = 0; t < 3 * nt; ++t)
      if (obj_tris[t] < 0 || obj_tris[t] >= nv) throw std::invalid_argument("lg_validate_batch: triangle index out of range");
    for (long long i = 0; i < n; ++i)
      if (grasps[i].n_contacts < 0 || grasps[i].n_contacts > LG_MAX_CONTACTS || grasps[i].dof < 0 ||
          grasps[i].dof > LG_MAX_DOF)
        throw std::invalid_argument("lg_validate_batch: grasp record out of range");
    Buf bg, bo, bv, bt, sc[6];
    const lg_grasp* d_g = dupload(bg, grasps, (size_t)n, s);
    lg_grasp_check* d_o = dalloc<lg_grasp_check>(bo, (size_t)n);
    ValCfg C;
    C.dof = hand->dof;
    C.contact_tol = p->contact_tol;
    C.penetration_margin = p->penetration_margin;
    C.lambda = p->lambda_torque;
    C.mu = p->mu;
    C.eps_stable = p->eps_stable;
    C.o.iterations = p->pgd_iterations;
    C.o.warm_iterations = p->pgd_warm_iterations;
    C.o.step = p->pgd_step;
    C.o.max_bt = 20;  // WrenchSolveOptions default (wrench.hpp)
    C.obj_v = nt ? dupload(bv, obj_verts, 3 * (size_t)nv, s) : nullptr;
    C.obj_t = nt ? dupload(bt, obj_tris, 3 * (size_t)nt, s) : nullptr;
    C.nt = nt;
    std::vector<double> col(ns);
    for (int a = 0; a < 6; ++a) {
      for (int i = 0; i < ns; ++i) col[i] = samples[6 * i + a];
      if (ns) dupload(sc[a], col.data(), (size_t)ns, s);
      CK(cudaStreamSynchronize(s));
    }
    DSamples S = make_samples(sc, ns);
    k_validate<<<(unsigned)n, 256, 0, s>>>(n, d_g, C, S, d_o);
    check_launch();
    k_validate_wrench<<<grid_for(n, 64), 64, 0, s>>>(n, d_g, C, d_o);
    check_launch();
    CK(cudaMemcpyAsync(out, d_o, sizeof(lg_grasp_check) * n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  });
}

int lg_collision_batch(lg_ctx* ctx, const lg_hand_desc* hand, int m, const double* q,
                       const double* poses, const double* samples, int n, double margin,
                       uint8_t* clean, double* max_penetration) {
  return lgc::guard([&] {
    if (!ctx || !hand || m < 0) throw std::invalid_argument("lg_collision_batch: bad argument");
    if (margin < 0.0) throw std::invalid_argument("broad_phase: negative margin");
    if (m == 0) return;
    use_ctx(ctx);
    cudaStream_t s = ctx->stream;
    bind_hand(ctx, *hand);
    std::vector<double> col(std::max(n, 1));
    Buf sc[6];
    for (int a = 0; a < 6; ++a) {
      for (int i = 0; i < n; ++i) col[i] = samples[6 * i + a];
      dupload(sc[a], col.data(), (size_t)std::max(n, 1), s);
      CK(cudaStreamSynchronize(s));
    }
    DSamples S = make_samples(sc, n);
    std::vector<double> qp((size_t)m * kMaxDof, 0.0);
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < hand->dof; ++j) qp[(size_t)i * kMaxDof + j] = q[(size_t)i * hand->dof + j];
    std::vector<int> ids(m), acc(m, 1);
    for (int i = 0; i < m; ++i) ids[i] = i;
    Buf bq, bp, bi, ba, bb, bc, bm;
    double* d_q = dupload(bq, qp.data(), qp.size(), s);
    double* d_p = dupload(bp, poses, (size_t)m * 12, s);
    int* d_i = dupload(bi, ids.data(), ids.size(), s);
    int* d_a = dupload(ba, acc.data(), acc.size(), s);
    double* d_b = dalloc<double>(bb, (size_t)m * 6);
    uint8_t* d_c = dalloc<uint8_t>(bc, (size_t)m);
    double* d_m = dalloc<double>(bm, (size_t)m);
    if (n > 0) {
      k_obj_aabb<<<m, 256, 0, s>>>(m, S, d_p, d_a, d_b);
      check_launch();
    }
    GridBufs gb;
    CollCfg cc;
    cc.margin = margin;
    cc.raw = S;
    cc.part_link = ctx->h_part_link.as<int>();
    cc.grid = build_grid(ctx, S, samples, n, 0.005, gb, s);
    coll_kernel(cc)<<<(m + kCollWarps - 1) / kCollWarps, 32 * kCollWarps, 0, s>>>(m, cc, d_i, nullptr, d_q,
                                                                             d_p, d_b, 0, d_c, d_m);
    check_launch();
    CK(cudaMemcpyAsync(clean, d_c, (size_t)m, cudaMemcpyDeviceToHost, s));
    if (max_penetration)
      CK(cudaMemcpyAsync(max_penetration, d_m, sizeof(double) * m, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  });
}

int lg_realize_batch(lg_ctx* ctx, const lg_hand_desc* hand, int m, const int* k,
                     const double* object_points, const double* object_normals, const int* links,
                     const double* hand_points, const double* hand_normals, double beta,
                     int iterations, double step_clamp, double residual_tol, double damping_scale,
                     int finetune_rounds, int finetune_iterations, double* q, double* max_residual,
                     int* finite, unsigned long long* used_joints) {
  return lgc::guard([&] {
    if (!ctx || !hand || m < 0) throw std::invalid_argument("lg_realize_batch: bad argument");
    if (beta <= 0.0) throw std::invalid_argument("solve_contact_ik: beta must be > 0");
    if (m == 0) return;
    use_ctx(ctx);
    cudaStream_t s = ctx->stream;
    bind_hand(ctx, *hand);
    std::vector<double> tg((size_t)m * kMaxK * 12, 0.0);
    std::vector<int> tl((size_t)m * kMaxK, 0);
    size_t off = 0;
    for (int i = 0; i < m; ++i) {
      if (k[i] < 1 || k[i] > kMaxK) throw std::invalid_argument("realize_grasp: 1..5 targets");
      for (int c = 0; c < k[i]; ++c, ++off) {
        if (links[off] < 0 || links[off] >= hand->n_links)
          throw std::invalid_argument("solve_contact_ik: invalid target link");
        double* T = &tg[((size_t)i * kMaxK + c) * 12];
        for (int a = 0; a < 3; ++a) {
          T[a] = object_points[3 * off + a];
          T[3 + a] = object_normals[3 * off + a];
          T[6 + a] = hand_points[3 * off + a];
          T[9 + a] = hand_normals[3 * off + a];
        }
        tl[(size_t)i * kMaxK + c] = links[off];
      }
    }
    std::vector<double> q0((size_t)m * kMaxDof, 0.0);
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < hand->dof; ++j) q0[(size_t)i * kMaxDof + j] = q[(size_t)i * hand->dof + j];
    Buf bk, bt, bl, bq, br, bf, bu;
    int* d_k = dupload(bk, k, (size_t)m, s);
    double* d_t = dupload(bt, tg.data(), tg.size(), s);
    int* d_l = dupload(bl, tl.data(), tl.size(), s);
    double* d_q = dupload(bq, q0.data(), q0.size(), s);
    double* d_r = dalloc<double>(br, (size_t)m);
    int* d_f = dalloc<int>(bf, (size_t)m);
    auto* d_u = dalloc<unsigned long long>(bu, (size_t)m);
    IkCfg P;
    P.beta = beta;
    P.step_clamp = step_clamp;
    P.residual_tol = residual_tol;
    P.damping_scale = damping_scale;
    P.damping_min = 1e-6;
    P.iterations = iterations;
    P.max_backtracks = 10;
    launch_realize_warp(s, m, 0, d_k, P, finetune_rounds, finetune_iterations, d_t, kMaxK * 12, d_l,
                        kMaxK, d_q, d_q, d_r, d_f, d_u, hand->dof, hand->n_links);
    check_launch();
    auto hq = ddownload(d_q, q0.size(), s);
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < hand->dof; ++j) q[(size_t)i * hand->dof + j] = hq[(size_t)i * kMaxDof + j];
    CK(cudaMemcpyAsync(max_residual, d_r, sizeof(double) * m, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(finite, d_f, sizeof(int) * m, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(used_joints, d_u, sizeof(unsigned long long) * m, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  });
}

int lg_contact_ik_batch(lg_ctx* ctx, const lg_hand_desc* hand, int m, const int* k,
                        const double* q0, const double* object_points, const double* object_normals,
                        const int* links, const double* hand_points, const double* hand_normals,
                        double beta, int iterations, double step_clamp, double residual_tol,
                        double damping_scale, double damping_min, int max_backtracks, double* q,
                        int* finite, unsigned long long* used_joints, int* iterations_out,
                        double* objective, double* position_residual, double* normal_cosine) {
  return lgc::guard([&] {
    if (!ctx || !hand || m < 0 || (m > 0 && (!k || !q0 || !q || !finite || !used_joints ||
                                             !iterations_out || !objective)))
      throw std::invalid_argument("lg_contact_ik_batch: bad argument");
    if (beta <= 0.0) throw std::invalid_argument("solve_contact_ik: beta must be > 0");
    if (m == 0) return;
    use_ctx(ctx);
    cudaStream_t s = ctx->stream;
    bind_hand(ctx, *hand);
    std::vector<double> tg((size_t)m * kMaxK * 12, 0.0);
    std::vector<int> tl((size_t)m * kMaxK, 0);
    size_t off = 0;
    for (int i = 0; i < m; ++i) {
      if (k[i] < 0 || k[i] > kMaxK)
        throw std::invalid_argument("solve_contact_ik: the device takes 0..5 targets");
      for (int c = 0; c < k[i]; ++c, ++off) {
        if (links[off] < 0 || links[off] >= hand->n_links)
          throw std::invalid_argument("solve_contact_ik: invalid target link");
        double* T = &tg[((size_t)i * kMaxK + c) * 12];
        for (int a = 0; a < 3; ++a) {
          T[a] = object_points[3 * off + a];
          T[3 + a] = object_normals[3 * off + a];
          T[6 + a] = hand_points[3 * off + a];
          T[9 + a] = hand_normals[3 * off + a];
        }
        for (int a = 0; a < 12; ++a)
          if (!std::isfinite(T[a])) throw std::invalid_argument("solve_contact_ik: non-finite target");
        tl[(size_t)i * kMaxK + c] = links[off];
      }
    }
    std::vector<double> qi((size_t)m * kMaxDof, 0.0);
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < hand->dof; ++j) qi[(size_t)i * kMaxDof + j] = q0[(size_t)i * hand->dof + j];
    Buf bk, bt, bl, bq, br, bf, bu, bit, bob, bpr, bco;
    int* d_k = dupload(bk, k, (size_t)m, s);
    double* d_t = dupload(bt, tg.data(), tg.size(), s);
    int* d_l = dupload(bl, tl.data(), tl.size(), s);
    double* d_q = dupload(bq, qi.data(), qi.size(), s);
    double* d_r = dalloc<double>(br, (size_t)m);
    int* d_f = dalloc<int>(bf, (size_t)m);
    auto* d_u = dalloc<unsigned long long>(bu, (size_t)m);
    IkOut io;
    io.iterations = dalloc<int>(bit, (size_t)m);
    io.objective = dalloc<double>(bob, (size_t)m);
    io.position = dalloc<double>(bpr, (size_t)m * kMaxK);
    io.cosine = dalloc<double>(bco, (size_t)m * kMaxK);
    IkCfg P;
    P.beta = beta;
    P.step_clamp = step_clamp;
    P.residual_tol = residual_tol;
    P.damping_scale = damping_scale;
    P.damping_min = damping_min;
    P.iterations = iterations;
    P.max_backtracks = max_backtracks;
    launch_realize_warp(s, m, 0, d_k, P, 0, 0, d_t, kMaxK * 12, d_l, kMaxK, d_q, d_q, d_r, d_f, d_u,
                        hand->dof, hand->n_links, &io);
    check_launch();
    auto hq = ddownload(d_q, qi.size(), s);
    auto hf = ddownload(d_f, (size_t)m, s);
    auto hu = ddownload(d_u, (size_t)m, s);
    auto hit = ddownload(io.iterations, (size_t)m, s);
    auto hob = ddownload(io.objective, (size_t)m, s);
    auto hpr = ddownload(io.position, (size_t)m * kMaxK, s);
    auto hco = ddownload(io.cosine, (size_t)m * kMaxK, s);
    off = 0;
    for (int i = 0; i < m; ++i) {
      for (int j = 0; j < hand->dof; ++j) q[(size_t)i * hand->dof + j] = hq[(size_t)i * kMaxDof + j];
      finite[i] = hf[i];
      used_joints[i] = hu[i];
      iterations_out[i] = hit[i];
      objective[i] = hob[i];
      for (int c = 0; c < k[i]; ++c, ++off) {
        if (position_residual) position_residual[off] = hpr[(size_t)i * kMaxK + c];
        if (normal_cosine) normal_cosine[off] = hco[(size_t)i * kMaxK + c];
      }
    }
  });
}

}  // extern "C"

// ================================================================= C-ABI
extern "C" {

const char* lg_version(void) {
  return "graspgen-b200 sm_100a fp64 (--fmad=false), lg_math canonical order";
}

int lg_device_count(int* n) {
  return lgc::guard([&] {
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) c = 0;
    *n = c;
  });
}

int lg_ctx_create(int device, lg_ctx** out) {
  return lgc::guard([&] {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
      throw lgc::cuda_error("no CUDA device available (the library has no CPU fallback)");
    if (device < 0 || device >= n) throw std::invalid_argument("lg_ctx_create: bad device index");
    CK(cudaSetDevice(device));
    auto* c = new lg_ctx;
    c->device = device;
    cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
      delete c;
      throw lgc::cuda_error(std::string("cudaStreamCreate: ") + cudaGetErrorString(e));
    }
    {
      std::lock_guard<std::mutex> lk(g_streams_mu);
      g_live_streams.insert(c->stream);
    }
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = ~0ull;  // keep freed blocks cached in the pool
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    *out = c;
  });
}

void lg_ctx_destroy(lg_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  for (Buf* b : {&ctx->h_vert_off, &ctx->h_verts, &ctx->h_tri_off, &ctx->h_tris, &ctx->h_plane_off,
                 &ctx->h_planes, &ctx->h_bounds, &ctx->h_part_link})
    b->release();
  if (ctx->cub_tmp) cudaFree(ctx->cub_tmp);
  if (ctx->stream) {
    cudaStreamSynchronize(ctx->stream);
    drop_cache(ctx->stream);
    {
      std::lock_guard<std::mutex> lk(g_streams_mu);
      g_live_streams.erase(ctx->stream);
    }
    cudaStreamDestroy(ctx->stream);
  }
  delete ctx;
}

int lg_field_build(lg_ctx* ctx, const lg_hand_desc* hand, const lg_patches_desc* patches, int N,
                   double w, uint64_t seed, int C, lg_field** out) {
  return lgc::guard([&] {
    if (!ctx || !hand || !patches || !out) throw std::invalid_argument("lg_field_build: null argument");
    use_ctx(ctx);
    auto f = std::make_unique<lg_field>();
    f->ctx = ctx;
    build_field_device(ctx, *hand, *patches, N, w, seed, C, f.get());
    *out = f.release();
  });
}

int lg_field_export(lg_field* f, lg_field_csr* o) {
  return lgc::guard([&] {
    if (!f || !o) throw std::invalid_argument("lg_field_export: null argument");
    use_ctx(f->ctx);
    export_field(f);
    const DField& F = f->f;
    o->box_width = F.w;
    o->codebook_size = F.C;
    o->codebook = f->x_codebook.data();
    o->n_patches = F.P;
    o->patch_link = f->x_patch_link.data();
    o->patch_box_off = f->x_patch_box_off.data();
    o->n_boxes = F.B;
    o->box_cell = f->x_box_cell.data();
    o->box_code_off = f->x_box_code_off.data();
    o->n_codes = f->n_codes;
    o->codes = f->x_codes.data();
    o->rep_link = f->x_rep_link.data();
    o->rep_point = f->x_rep_point.data();
    o->rep_normal = f->x_rep_normal.data();
    o->n_vectors = f->n_vectors;
  });
}

int lg_field_save(lg_field* f, const char* path, uint64_t key) {
  return lgc::guard([&] {
    if (!f || !path) throw std::invalid_argument("lg_field_save: null argument");
    use_ctx(f->ctx);
    save_field(f, path, key);
  });
}

int lg_field_load(lg_ctx* ctx, const lg_hand_desc* hand, const char* path, uint64_t key,
                  lg_field** out) {
  return lgc::guard([&] {
    if (!ctx || !hand || !path || !out) throw std::invalid_argument("lg_field_load: null argument");
    use_ctx(ctx);
    *out = nullptr;
    auto f = std::make_unique<lg_field>();
    f->ctx = ctx;
    if (load_field(ctx, *hand, path, key, f.get())) *out = f.release();
  });
}

void lg_field_destroy(lg_field* f) { delete f; }

int lg_query_domains_batch(lg_ctx* ctx, lg_field* f, const int* group_of_patch,
                           const double* samples, int n, const double* poses, int m, double theta,
                           uint32_t* masks, double* scores) {
  return lgc::guard([&] {
    if (!ctx || !f || !samples || !poses || !masks) throw std::invalid_argument("lg_query_domains_batch: null argument");
    use_ctx(ctx);
    cudaStream_t s = ctx->stream;
    std::vector<double> col(n);
    Buf sc[6];
    for (int a = 0; a < 6; ++a) {
      for (int i = 0; i < n; ++i) col[i] = samples[6 * i + a];
      dupload(sc[a], col.data(), (size_t)n, s);
      CK(cudaStreamSynchronize(s));
    }
    DSamples S = make_samples(sc, n);
    Buf bp, bg, bm, bc, ba;
    double* d_pose = dupload(bp, poses, 12 * (size_t)m, s);
    int* d_g = dupload(bg, group_of_patch, (size_t)f->f.P, s);
    uint32_t* d_mask = dalloc<uint32_t>(bm, (size_t)m * n);
    std::vector<int> acc(m, 1);
    int* d_acc = dupload(ba, acc.data(), acc.size(), s);
    int G = 0;
    for (int p = 0; p < f->f.P; ++p) G = std::max(G, group_of_patch[p] + 1);
    int* d_cnt = dalloc<int>(bc, (size_t)m * std::max(G, 1));
    DField fq = f->f;  // the dense path bakes the field's own groups into rec
    if (!std::equal(f->h_gop.begin(), f->h_gop.end(), group_of_patch)) fq.grid_ok = 0;
    if (fq.grid_ok && ensure_dirlists(f, theta)) {
      size_t qsm = codebook_smem(k_query3, f->f.C);
      k_query3<<<m, 256, qsm, s>>>(m, f->f, S, d_pose, d_acc, theta, G, qsm > 0, d_mask, d_cnt);
    } else {
      size_t qsm = codebook_smem(k_query, f->f.C);
      k_query<<<m, 256, qsm, s>>>(m, fq, d_g, S, d_pose, d_acc, theta, G, qsm > 0, d_mask, d_cnt);
    }
    check_launch();
    CK(cudaMemcpyAsync(masks, d_mask, sizeof(uint32_t) * m * n, cudaMemcpyDeviceToHost, s));
    if (scores) {
      Buf bsc;
      double* d_sc = dalloc<double>(bsc, (size_t)m * n);
      k_query_scores<<<m, 256, 0, s>>>(m, f->f, d_g, S, d_pose, theta, d_sc);
      check_launch();
      CK(cudaMemcpyAsync(scores, d_sc, sizeof(double) * m * n, cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));
  });
}

int lg_preprocess(lg_ctx* ctx, const double* samples, int n, double h, double d, uint8_t* keep) {
  return lgc::guard([&] {
    if (h <= 0.0 || d < 0.0) throw std::invalid_argument("preprocess_object: bad probe dimensions");
    use_ctx(ctx);
    cudaStream_t s = ctx->stream;
    std::vector<double> col(n);
    Buf sc[6], bk;
    for (int a = 0; a < 6; ++a) {
      for (int i = 0; i < n; ++i) col[i] = samples[6 * i + a];
      dupload(sc[a], col.data(), (size_t)n, s);
      CK(cudaStreamSynchronize(s));
    }
    uint8_t* d_keep = dalloc<uint8_t>(bk, (size_t)n);
    const DSamples S = make_samples(sc, n);
    GridBufs gb;
    const DGrid g = build_grid(ctx, S, samples, n, 0.5 * h, gb, s);
    preprocess_device(ctx, S, g, h, d, d_keep, s);
    CK(cudaMemcpyAsync(keep, d_keep, n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  });
}

namespace lgd {
// The hot path's transcendentals (csrc/lg_libm.h) evaluated on the device, for
// the bit-exactness check against the host glibc (tests/test_libm.py).
__global__ void k_libm_eval(int which, int n, const double* x, const double* y, double* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double a = x[i], r;
    switch (which) {
      case 0: r = lgm::xsin(a); break;
      case 1: r = lgm::xcos(a); break;
      case 2: r = lgm::xlog(a); break;
      case 3: r = lgm::xatan2(a, y[i]); break;
      default: r = lgm::xhypot(a, y[i]); break;
    }
    out[i] = r;
  }
}
}  // namespace lgd

long long lg_debug_canary_violations(void) { return g_canary_bad.load(); }

int lg_libm_eval(lg_ctx* ctx, int which, long long n, const double* x, const double* y,
                 double* out) {
  return lgc::guard([&] {
    if (!ctx || !x || !out || n < 0 || which < 0 || which > 4 || (which >= 3 && !y))
      throw std::invalid_argument("lg_libm_eval: bad argument");
    use_ctx(ctx);
    cudaStream_t s = ctx->stream;
    Buf bx, by, bo;
    dupload(bx, x, (size_t)n, s);
    if (which >= 3) dupload(by, y, (size_t)n, s);
    double* d_out = dalloc<double>(bo, (size_t)n);
    lgd::k_libm_eval<<<grid_for((int)n, 256), 256, 0, s>>>(which, (int)n, (const double*)bx.p,
                                                           which >= 3 ? (const double*)by.p : nullptr,
                                                           d_out);
    check_launch();
    LAUNCH(ctx);
    CK(cudaMemcpyAsync(out, d_out, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  });
}

int lg_run_batch_field(lg_ctx* ctx, const lg_hand_desc* hand, const lg_patches_desc* patches,
                       lg_field* field, const double* raw, int n_raw, const lg_run_params* p,
                       lg_result** out) {
  return lgc::guard([&] {
    if (!ctx || !hand || !patches || !raw || !p || !out) throw std::invalid_argument("lg_run_batch: null argument");
    use_ctx(ctx);
    auto r = std::make_unique<lg_result>();
    run_batch_device(ctx, *hand, *patches, field, raw, n_raw, *p, r->r);
    *out = r.release();
  });
}

int lg_run_batch(lg_ctx* ctx, const lg_hand_desc* hand, const lg_patches_desc* patches,
                 const double* raw, int n_raw, const lg_run_params* p, lg_result** out) {
  return lg_run_batch_field(ctx, hand, patches, nullptr, raw, n_raw, p, out);
}

int lg_result_profile(const lg_result* r, lg_profile* out) {
  return lgc::guard([&] {
    if (!r || !out) throw std::invalid_argument("lg_result_profile: null argument");
    *out = r->r.profile;
  });
}
long long lg_result_num_grasps(const lg_result* r) { return r ? (long long)r->r.grasps.size() : 0; }
const lg_grasp* lg_result_grasps(const lg_result* r) { return r ? r->r.grasps.data() : nullptr; }
long long lg_result_num_traces(const lg_result* r) { return r ? (long long)r->r.traces.size() : 0; }
const lg_trace* lg_result_traces(const lg_result* r) { return r ? r->r.traces.data() : nullptr; }
void lg_result_destroy(lg_result* r) { delete r; }

}  // extern "C"

// ===================================================================== multi-GPU
// Seed sharding: rank r of R runs lg_run_batch with
// shard_rank = r, shard_count = R on its own GPU (every per-candidate RNG
// stream depends only on (seed, tag, c or g), so the shards are independent
// and the union is the single-GPU result).  The only collective is the final
// gather of the kept grasps to rank 0 over NCCL: one ncclAllGather of a fixed
// per-rank header (grasp count, funnel counters, stage times), then grouped
// ncclSend / ncclRecv of the packed lg_grasp records to rank 0, which orders
// them by g = pass*batch + c — run_batch's `kept` order (pipeline.cpp:607-614).
// This replaces the reference's only parallelism, parallel_for over chunks of
// candidates (parallel.hpp:24-56, pipeline.cpp:382-391).
//
// NCCL is bound at run time (dlopen of libnccl.so.2, reusing an already-loaded
// copy such as the one PyTorch brings), so the library has no link-time NCCL
// dependency and single-GPU callers never load it.
#include <dlfcn.h>
#include <nccl.h>

namespace {
struct NcclApi {
  void* h = nullptr;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclAllGather) allGather = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclGetErrorString) errorString = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.h = h;
    api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
    api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
    api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
    api.allGather = (decltype(api.allGather))dlsym(h, "ncclAllGather");
    api.send = (decltype(api.send))dlsym(h, "ncclSend");
    api.recv = (decltype(api.recv))dlsym(h, "ncclRecv");
    api.groupStart = (decltype(api.groupStart))dlsym(h, "ncclGroupStart");
    api.groupEnd = (decltype(api.groupEnd))dlsym(h, "ncclGroupEnd");
    api.errorString = (decltype(api.errorString))dlsym(h, "ncclGetErrorString");
  });
  if (!api.h || !api.commInitRank || !api.allGather || !api.send || !api.recv)
    throw lgc::cuda_error("NCCL (libnccl.so.2) is not available");
  return api;
}

void NK(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw lgc::cuda_error(std::string(what) + ": " +
                          (nccl().errorString ? nccl().errorString(r) : "NCCL error"));
}

// Per-rank header exchanged by the all-gather (int64 slots; doubles bit-cast).
enum : int {
  kHdrGrasps = 0, kHdrCandidates, kHdrPlaced, kHdrBalanced, kHdrIkFinite, kHdrPenFree,
  kHdrIkConv, kHdrStable, kHdrValid, kHdrLaunches, kHdrDevSec, kHdrTotal, kHdrPlacementS,
  kHdrContactS, kHdrKinS, kHdrPostS, kHdrFieldS, kHdrN = 20
};
long long dbits(double v) {
  long long b;
  std::memcpy(&b, &v, 8);
  return b;
}
double bitsd(long long b) {
  double v;
  std::memcpy(&v, &b, 8);
  return v;
}
}  // namespace

struct lg_comm {
  lg_ctx* ctx = nullptr;
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  std::vector<lg_grasp> merged;
};

extern "C" {

int lg_comm_unique_id(unsigned char* id) {
  return lgc::guard([&] {
    if (!id) throw std::invalid_argument("lg_comm_unique_id: null argument");
    static_assert(sizeof(ncclUniqueId) == LG_COMM_ID_BYTES, "NCCL unique id size");
    ncclUniqueId u;
    NK(nccl().getUniqueId(&u), "ncclGetUniqueId");
    std::memcpy(id, &u, sizeof(u));
  });
}

int lg_comm_init(lg_ctx* ctx, const unsigned char* id, int rank, int world, lg_comm** out) {
  return lgc::guard([&] {
    if (!ctx || !id || !out || world < 1 || rank < 0 || rank >= world)
      throw std::invalid_argument("lg_comm_init: bad argument");
    use_ctx(ctx);
    auto c = std::make_unique<lg_comm>();
    c->ctx = ctx;
    c->rank = rank;
    c->world = world;
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    NK(nccl().commInitRank(&c->comm, world, u, rank), "ncclCommInitRank");
    *out = c.release();
  });
}

void lg_comm_destroy(lg_comm* c) {
  if (!c) return;
  if (c->comm && nccl().commDestroy) nccl().commDestroy(c->comm);
  delete c;
}

int lg_comm_gather(lg_comm* c, const lg_grasp* grasps, long long n, const lg_profile* profile,
                   const lg_grasp** all, long long* n_all, lg_profile* merged) {
  return lgc::guard([&] {
    if (!c || (!grasps && n) || !profile || !all || !n_all)
      throw std::invalid_argument("lg_comm_gather: null argument");
    use_ctx(c->ctx);
    cudaStream_t s = c->ctx->stream;
    NcclApi& api = nccl();
    const int R = c->world;
    // 1. headers
    std::vector<long long> hdr(kHdrN, 0);
    const lg_profile& p = *profile;
    hdr[kHdrGrasps] = n;
    hdr[kHdrCandidates] = p.candidates;
    hdr[kHdrPlaced] = p.placements_accepted;
    hdr[kHdrBalanced] = p.contact_sets_balanced;
    hdr[kHdrIkFinite] = p.ik_finite;
    hdr[kHdrPenFree] = p.penetration_free;
    hdr[kHdrIkConv] = p.ik_converged;
    hdr[kHdrStable] = p.stable;
    hdr[kHdrValid] = p.valid;
    hdr[kHdrLaunches] = p.gpu_launches;
    hdr[kHdrDevSec] = dbits(p.device_seconds);
    hdr[kHdrTotal] = dbits(p.total);
    hdr[kHdrPlacementS] = dbits(p.placement_domains);
    hdr[kHdrContactS] = dbits(p.contact_optimization);
    hdr[kHdrKinS] = dbits(p.kinematics_optimization);
    hdr[kHdrPostS] = dbits(p.postprocessing);
    hdr[kHdrFieldS] = dbits(p.field_build);
    Buf bh, ba;
    long long* d_h = dupload(bh, hdr.data(), hdr.size(), s);
    long long* d_all = dalloc<long long>(ba, (size_t)kHdrN * R);
    NK(api.allGather(d_h, d_all, kHdrN, ncclInt64, c->comm, s), "ncclAllGather");
    std::vector<long long> H = ddownload(d_all, (size_t)kHdrN * R, s);
    // 2. records to rank 0
    const size_t rec = sizeof(lg_grasp);
    std::vector<long long> off(R + 1, 0);
    for (int r = 0; r < R; ++r) off[r + 1] = off[r] + H[(size_t)r * kHdrN + kHdrGrasps];
    Buf bs, br;
    uint8_t* d_send = nullptr;
    uint8_t* d_recv = nullptr;
    if (c->rank != 0 && n > 0) d_send = dupload(bs, (const uint8_t*)grasps, (size_t)n * rec, s);
    if (c->rank == 0 && off[R] - n > 0) d_recv = dalloc<uint8_t>(br, (size_t)(off[R] - n) * rec);
    NK(api.groupStart(), "ncclGroupStart");
    if (c->rank == 0) {
      for (int r = 1; r < R; ++r) {
        long long cnt = off[r + 1] - off[r];
        if (cnt > 0)
          NK(api.recv(d_recv + (size_t)(off[r] - n) * rec, (size_t)cnt * rec, ncclUint8, r, c->comm, s),
             "ncclRecv");
      }
    } else if (n > 0) {
      NK(api.send(d_send, (size_t)n * rec, ncclUint8, 0, c->comm, s), "ncclSend");
    }
    NK(api.groupEnd(), "ncclGroupEnd");
    CK(cudaStreamSynchronize(s));
    if (c->rank != 0) {
      *all = nullptr;
      *n_all = 0;
      if (merged) std::memset(merged, 0, sizeof(*merged));
      return;
    }
    // 3. merge on rank 0: kept order = ascending g (stable)
    c->merged.assign(grasps, grasps + n);
    if (off[R] > n) {
      std::vector<uint8_t> h = ddownload(d_recv, (size_t)(off[R] - n) * rec, s);
      const lg_grasp* g = (const lg_grasp*)h.data();
      c->merged.insert(c->merged.end(), g, g + (off[R] - n));
    }
    std::stable_sort(c->merged.begin(), c->merged.end(),
                     [](const lg_grasp& a, const lg_grasp& b) { return a.g < b.g; });
    *all = c->merged.data();
    *n_all = (long long)c->merged.size();
    if (merged) {
      *merged = p;
      auto sum = [&](int k) {
        long long t = 0;
        for (int r = 0; r < R; ++r) t += H[(size_t)r * kHdrN + k];
        return t;
      };
      auto mx = [&](int k) {
        double t = 0.0;
        for (int r = 0; r < R; ++r) t = std::max(t, bitsd(H[(size_t)r * kHdrN + k]));
        return t;
      };
      merged->candidates = sum(kHdrCandidates);
      merged->placements_accepted = sum(kHdrPlaced);
      merged->contact_sets_balanced = sum(kHdrBalanced);
      merged->ik_finite = sum(kHdrIkFinite);
      merged->penetration_free = sum(kHdrPenFree);
      merged->ik_converged = sum(kHdrIkConv);
      merged->stable = sum(kHdrStable);
      merged->valid = sum(kHdrValid);
      merged->gpu_launches = sum(kHdrLaunches);
      merged->device_seconds = mx(kHdrDevSec);
      merged->total = mx(kHdrTotal);
      merged->placement_domains = mx(kHdrPlacementS);
      merged->contact_optimization = mx(kHdrContactS);
      merged->kinematics_optimization = mx(kHdrKinS);
      merged->postprocessing = mx(kHdrPostS);
      merged->field_build = mx(kHdrFieldS);
      merged->grasps_per_second = merged->total > 0.0 ? merged->valid / merged->total : 0.0;
    }
  });
}

}  // extern "C"

// ================================================== stage-level entry points
// The reference's public hot-path functions, batched:
// place_object, query_domains (full ContactDomain elements with hits),
// reverse_lookup, optimize_contacts, realize_grasp's final projection, and
// validate_grasp_collisions' full report.  Each reuses the kernels of
// run_batch; the parity tests call them against the reference's own
// functions (oracle/_ref) on identical inputs.
namespace lgd {

// query_domains (contact_field.cpp:380-448), one pose: pass 1 counts each
// sample's hits per dependency group, pass 2 writes the elements.
__global__ void k_qe_count(int n, DField f, DSamples S, Xf x, double theta, const int* gop, int G,
                           int* cnt) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  V3 p = xf_apply(x, S.p(i)), nn = xf_rotate(x, S.nrm(i));
  sample_hits(f, f.codebook, p, nn, theta, [&](int patch, int, double) {
    int g = gop[patch];
    if (g >= 0 && g < G) ++cnt[(size_t)g * n + i];
  });
}

__global__ void k_qe_fill(int n, DField f, DSamples S, Xf x, double theta, const int* gop, int G,
                          const long long* elem_of, const long long* hit_of, long long* hit_off,
                          int* sample, double* pos, double* nrm, double* score, int* hit_patch,
                          int* hit_box) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  V3 p = xf_apply(x, S.p(i)), nn = xf_rotate(x, S.nrm(i));
  for (int g = 0; g < G; ++g) {
    long long e = elem_of[(size_t)g * n + i];
    if (e < 0) continue;
    long long h = hit_of[(size_t)g * n + i];
    hit_off[e] = h;
    sample[e] = i;
    v3_store(pos + 3 * e, p);
    v3_store(nrm + 3 * e, nn);
    double sc = 0.0;  // DomainElement::score starts at 0.0 (contact_field.hpp:104)
    sample_hits(f, f.codebook, p, nn, theta, [&](int patch, int b, double) {
      if (gop[patch] != g) return;
      double best = -2.0;
      for (long long q = f.box_code_off[b]; q < f.box_code_off[b + 1]; ++q) {
        int c = f.codes[q];
        best = dmax(best, -dot(v3(f.codebook[3 * c], f.codebook[3 * c + 1], f.codebook[3 * c + 2]), nn));
      }
      sc = dmax(sc, best);
      hit_patch[h] = patch;
      hit_box[h] = b - f.patch_box_off[patch];
      ++h;
    });
    score[e] = sc;
  }
}

// reverse_lookup (contact_field.cpp:450-484) per element.
__global__ void k_reverse_lookup(int m, DField f, const long long* hit_off, const int* hit_patch,
                                 const int* hit_box, const double* nrm, const uint64_t* seeds,
                                 int* link, double* point, double* normal, int* err) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  long long h0 = hit_off[t], nh = hit_off[t + 1] - h0;
  if (nh <= 0) {
    atomicMax(err, 1);
    return;
  }
  DRng rng;
  rng.seed(seeds[t]);
  long long pick = (long long)rng.index((uint64_t)nh);
  int patch = hit_patch[h0 + pick], box = hit_box[h0 + pick];
  if (patch < 0 || patch >= f.P || box < 0 || box >= f.patch_box_off[patch + 1] - f.patch_box_off[patch]) {
    atomicMax(err, 2);
    return;
  }
  long long b = f.patch_box_off[patch] + box;
  V3 n = v3_load(nrm + 3 * t);
  int best = -1;
  double best_dot = -2.0;
  long long q0 = f.box_code_off[b], q1 = f.box_code_off[b + 1];
  for (long long q = q0; q < q1; ++q) {
    int c = f.codes[q];
    double d = -dot(v3(f.codebook[3 * c], f.codebook[3 * c + 1], f.codebook[3 * c + 2]), n);
    if (d > best_dot) {
      best_dot = d;
      best = (int)(q - q0);
    }
  }
  const double* rp = f.rep_pn + 6 * (q0 + best);
  v3_store(point + 3 * t, v3_load(rp));
  v3_store(normal + 3 * t, v3_load(rp + 3));
  link[t] = f.rep_link[q0 + best];
}

// optimize_contacts' stream draws from explicit seeds (contact_opt.cpp:61).
__global__ void k_copt_draws_seeded(int m, const uint64_t* seeds, long long per_cand, uint64_t* out) {
  int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= m) return;
  Mt64 g;
  mt_seed(g, seeds[a]);
  uint64_t* o = out + (size_t)a * per_cand;
  for (long long d = 0; d < per_cand; ++d) o[d] = mt_next(g);
}

// realize_grasp's final projection (pipeline.cpp:196-221, 250): realized
// contact and position residual per target at configuration q.
__global__ void k_realized(int m, int kmax, const int* k, const double* q, int dof, const int* links,
                           const double* obj_p, double* rp, double* rn, int* rl, double* res) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m * kmax) return;
  int i = t / kmax, c = t % kmax;
  if (c >= k[i]) return;
  double qq[kMaxDof];
  for (int j = 0; j < dof; ++j) qq[j] = q[(size_t)i * dof + j];
  Xf frames[kMaxLinks];
  fk(qq, frames);
  int l = links[t];
  Xf inv = xf_inverse(frames[l]);
  V3 sp = v3(0, 0, 0), sn = v3(0, 0, 0);
  double d = closest_on_parts(l, xf_apply(inv, v3_load(obj_p + 3 * t)), &sp, &sn);
  v3_store(rp + 3 * t, xf_apply(frames[l], sp));
  v3_store(rn + 3 * t, xf_rotate(frames[l], sn));
  rl[t] = l;
  res[t] = d;
}

// validate_grasp_collisions (collision.cpp:230-288), the full report: thread
// per configuration, violations deduplicated per link pair in pair order.
__global__ void k_collision_report(int m, const double* q, int dof, const double* poses, DSamples S,
                                   double margin, const int* part_link, int cap, int* n_viol,
                                   int* va, int* vb, double* vd, double* max_pen, int* pairs) {
  // pairs[3i..3i+2] = broad_pairs, narrow_gjk, narrow_halfplane (collision.hpp:57-65)
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  double qq[kMaxDof];
  for (int j = 0; j < dof; ++j) qq[j] = q[(size_t)i * dof + j];
  Xf frames[kMaxLinks];
  fk(qq, frames);
  Xf op = load_xf(poses + 12 * i);
  V3 omn = v3(kInf, kInf, kInf), omx = v3(-kInf, -kInf, -kInf);
  for (int s = 0; s < S.n; ++s) {
    V3 w = xf_apply(op, S.p(s));
    omn = vmin(omn, w);
    omx = vmax(omx, w);
  }
  const bool has_obj = S.n > 0;
  omn = v3(omn.x - margin, omn.y - margin, omn.z - margin);
  omx = v3(omx.x + margin, omx.y + margin, omx.z + margin);
  const int np = c_hand.n_parts;
  int nv = 0, npairs = 0, ngjk = 0, nhp = 0;
  double mp = 0.0;
  int* A = va + (size_t)i * cap;
  int* Bv = vb + (size_t)i * cap;
  double* D = vd + (size_t)i * cap;
  auto record = [&](int la, int lb, double depth) {
    for (int v = 0; v < nv && v < cap; ++v)
      if (A[v] == la && Bv[v] == lb) {
        D[v] = dmax(D[v], depth);
        return;
      }
    if (nv < cap) {
      A[nv] = la;
      Bv[nv] = lb;
      D[nv] = depth;
    }
    ++nv;
  };
  for (int a = 0; a < np; ++a) {
    const int la = part_link[a];
    V3 amn, amx;
    world_bounds(a, frames[la], &amn, &amx);
    amn = v3(amn.x - margin, amn.y - margin, amn.z - margin);
    amx = v3(amx.x + margin, amx.y + margin, amx.z + margin);
    for (int b = a + 1; b < np; ++b) {
      const int lb = part_link[b];
      V3 bmn, bmx;
      world_bounds(b, frames[lb], &bmn, &bmx);
      bmn = v3(bmn.x - margin, bmn.y - margin, bmn.z - margin);
      bmx = v3(bmx.x + margin, bmx.y + margin, bmx.z + margin);
      const bool ov = amn.x <= bmx.x && amn.y <= bmx.y && amn.z <= bmx.z && amx.x >= bmn.x &&
                      amx.y >= bmn.y && amx.z >= bmn.z;
      if (!ov) continue;
      ++npairs;
      if (la == lb || c_hand.parent[la] == lb || c_hand.parent[lb] == la) continue;
      ++ngjk;
      if (gjk_distance(a, frames[la], b, frames[lb]) == 0.0) record(la < lb ? la : lb, la < lb ? lb : la, 0.0);
    }
    if (has_obj && amn.x <= omx.x && amn.y <= omx.y && amn.z <= omx.z && amx.x >= omn.x &&
        amx.y >= omn.y && amx.z >= omn.z) {
      ++npairs;
      ++nhp;
      // object_penetration (collision.cpp:209-228)
      Xf inv = xf_inverse(frames[la]);
      const double* bb = c_hand.bounds + 6 * a;
      double md = 0.0;
      bool off = false;
      for (int s = 0; s < S.n; ++s) {
        V3 local = xf_apply(inv, xf_apply(op, S.p(s)));
        if (!(local.x >= bb[0] - 1e-9 && local.y >= bb[1] - 1e-9 && local.z >= bb[2] - 1e-9 &&
              local.x <= bb[3] + 1e-9 && local.y <= bb[4] + 1e-9 && local.z <= bb[5] + 1e-9))
          continue;
        double depth = part_interior_depth(a, local);
        if (depth > margin) {
          off = true;
          md = dmax(md, depth);
        }
      }
      if (off) {
        record(la, -1, md);
        mp = dmax(mp, md);
      }
    }
  }
  n_viol[i] = nv;
  max_pen[i] = mp;
  pairs[3 * i] = npairs;
  pairs[3 * i + 1] = ngjk;
  pairs[3 * i + 2] = nhp;
}

}  // namespace lgd

struct lg_domains {
  int n_groups = 0;
  std::vector<long long> group_off;  // [G+1] element ranges per group
  std::vector<long long> hit_off;    // [E+1]
  std::vector<int> sample, hit_patch, hit_box;
  std::vector<double> pos, nrm, score;
};

extern "C" {

int lg_query_domains_elements(lg_ctx* ctx, lg_field* f, const int* group_of_patch, int n_groups,
                              const double* samples, int n, const double* pose, double theta_hit,
                              lg_domains** out) {
  return lgc::guard([&] {
    if (!ctx || !f || !group_of_patch || !samples || !pose || !out || n < 0 || n_groups < 0)
      throw std::invalid_argument("lg_query_domains_elements: bad argument");
    for (int p = 0; p < f->f.P; ++p)
      if (group_of_patch[p] >= n_groups)
        throw std::invalid_argument("query_domains: index link out of range");
    use_ctx(ctx);
    cudaStream_t s = ctx->stream;
    auto d = std::make_unique<lg_domains>();
    d->n_groups = n_groups;
    const int G = n_groups;
    std::vector<double> col((size_t)std::max(n, 1));
    Buf sc[6], bg, bc;
    for (int a = 0; a < 6; ++a) {
      for (int i = 0; i < n; ++i) col[i] = samples[6 * i + a];
      dupload(sc[a], col.data(), (size_t)n, s);
      CK(cudaStreamSynchronize(s));
    }
    DSamples S = make_samples(sc, n);
    Xf x = lgm::xf_identity();
    x.R = lgm::m3_load(pose);
    x.t = lgm::v3_load(pose + 9);
    int* d_g = dupload(bg, group_of_patch, (size_t)f->f.P, s);
    int* d_c = dalloc<int>(bc, (size_t)std::max(G, 1) * std::max(n, 1));
    CK(cudaMemsetAsync(d_c, 0, sizeof(int) * (size_t)std::max(G, 1) * std::max(n, 1), s));
    d->group_off.assign((size_t)G + 1, 0);
    d->hit_off.assign(1, 0);
    if (n > 0 && G > 0) {
      lgd::k_qe_count<<<grid_for(n, 128), 128, 0, s>>>(n, f->f, S, x, theta_hit, d_g, G, d_c);
      check_launch();
      LAUNCH(ctx);
      auto cnt = ddownload(d_c, (size_t)G * n, s);
      std::vector<long long> eo((size_t)G * n, -1), ho((size_t)G * n, 0);
      long long E = 0, H = 0;
      for (int g = 0; g < G; ++g) {
        for (int i = 0; i < n; ++i) {
          int c = cnt[(size_t)g * n + i];
          if (!c) continue;
          eo[(size_t)g * n + i] = E++;
          ho[(size_t)g * n + i] = H;
          H += c;
        }
        d->group_off[g + 1] = E;
      }
      d->hit_off.assign((size_t)E + 1, H);
      d->sample.resize(E);
      d->pos.resize(3 * E);
      d->nrm.resize(3 * E);
      d->score.resize(E);
      d->hit_patch.resize(H);
      d->hit_box.resize(H);
      if (E > 0) {
        Buf be, bh, bho, bs, bp, bn, bsc, bhp, bhb;
        long long* d_eo = dupload(be, eo.data(), eo.size(), s);
        long long* d_ho = dupload(bh, ho.data(), ho.size(), s);
        long long* d_hoff = dalloc<long long>(bho, (size_t)E);
        int* d_s = dalloc<int>(bs, (size_t)E);
        double* d_p = dalloc<double>(bp, 3 * (size_t)E);
        double* d_n = dalloc<double>(bn, 3 * (size_t)E);
        double* d_sc = dalloc<double>(bsc, (size_t)E);
        int* d_hp = dalloc<int>(bhp, (size_t)H);
        int* d_hb = dalloc<int>(bhb, (size_t)H);
        lgd::k_qe_fill<<<grid_for(n, 128), 128, 0, s>>>(n, f->f, S, x, theta_hit, d_g, G, d_eo, d_ho,
                                                       d_hoff, d_s, d_p, d_n, d_sc, d_hp, d_hb);
        check_launch();
        LAUNCH(ctx);
        auto hoff = ddownload(d_hoff, (size_t)E, s);
        std::copy(hoff.begin(), hoff.end(), d->hit_off.begin());
        d->sample = ddownload(d_s, (size_t)E, s);
        d->pos = ddownload(d_p, 3 * (size_t)E, s);
        d->nrm = ddownload(d_n, 3 * (size_t)E, s);
        d->score = ddownload(d_sc, (size_t)E, s);
        d->hit_patch = ddownload(d_hp, (size_t)H, s);
        d->hit_box = ddownload(d_hb, (size_t)H, s);
      }
    }
    *out = d.release();
  });
}

int lg_domains_group(const lg_domains* d, int group, long long* first, long long* count) {
  return lgc::guard([&] {
    if (!d || group < 0 || group >= d->n_groups || !first || !count)
      throw std::invalid_argument("lg_domains_group: bad argument");
    *first = d->group_off[group];
    *count = d->group_off[group + 1] - d->group_off[group];
  });
}

int lg_domains_elements(const lg_domains* d, long long* n_elements, const int** sample,
                        const double** pos, const double** nrm, const double** score,
                        const long long** hit_off, const int** hit_patch, const int** hit_box) {
  return lgc::guard([&] {
    if (!d) throw std::invalid_argument("lg_domains_elements: null handle");
    if (n_elements) *n_elements = (long long)d->sample.size();
    if (sample) *sample = d->sample.data();
    if (pos) *pos = d->pos.data();
    if (nrm) *nrm = d->nrm.data();
    if (score) *score = d->score.data();
    if (hit_off) *hit_off = d->hit_off.data();
    if (hit_patch) *hit_patch = d->hit_patch.data();
    if (hit_box) *hit_box = d->hit_box.data();
  });
}

void lg_domains_destroy(lg_domains* d) { delete d; }

int lg_reverse_lookup_batch(lg_ctx* ctx, lg_field* f, int m, const long long* hit_off,
                            const int* hit_patch, const int* hit_box, const double* normals,
                            const uint64_t* seeds, int* link, double* point, double* normal) {
  return lgc::guard([&] {
    if (!ctx || !f || m < 0 || (m && (!hit_off || !normals || !seeds || !link || !point || !normal)))
      throw std::invalid_argument("lg_reverse_lookup_batch: bad argument");
    if (m == 0) return;
    use_ctx(ctx);
    cudaStream_t s = ctx->stream;
    const long long H = hit_off[m] - hit_off[0];
    Buf bo, bp, bb, bn, bs, bl, bpt, bnr, be;
    std::vector<long long> off(hit_off, hit_off + m + 1);
    for (auto& o : off) o -= hit_off[0];
    long long* d_o = dupload(bo, off.data(), off.size(), s);
    int* d_p = dupload(bp, hit_patch ? hit_patch + hit_off[0] : nullptr, (size_t)H, s);
    int* d_b = dupload(bb, hit_box ? hit_box + hit_off[0] : nullptr, (size_t)H, s);
    double* d_n = dupload(bn, normals, 3 * (size_t)m, s);
    uint64_t* d_s = dupload(bs, seeds, (size_t)m, s);
    int* d_l = dalloc<int>(bl, (size_t)m);
    double* d_pt = dalloc<double>(bpt, 3 * (size_t)m);
    double* d_nr = dalloc<double>(bnr, 3 * (size_t)m);
    int zero = 0;
    int* d_e = dupload(be, &zero, 1, s);
    lgd::k_reverse_lookup<<<grid_for(m, 128), 128, 0, s>>>(m, f->f, d_o, d_p, d_b, d_n, d_s, d_l, d_pt,
                                                          d_nr, d_e);
    check_launch();
    LAUNCH(ctx);
    int err = ddownload(d_e, 1, s)[0];
    if (err == 1) throw std::out_of_range("reverse_lookup: element has no hits");
    if (err == 2) throw std::out_of_range("reverse_lookup: stale element");
    auto l = ddownload(d_l, (size_t)m, s);
    auto pt = ddownload(d_pt, 3 * (size_t)m, s);
    auto nr = ddownload(d_nr, 3 * (size_t)m, s);
    std::copy(l.begin(), l.end(), link);
    std::copy(pt.begin(), pt.end(), point);
    std::copy(nr.begin(), nr.end(), normal);
  });
}

int lg_place_batch(lg_ctx* ctx, const lg_hand_desc* hand, const lg_patches_desc* patches,
                   lg_field* field, const double* raw, int n_raw, const lg_run_params* p, int c0,
                   int m, double* pose, int* accepted, double* penetration, int* n_static,
                   double* static_p, double* static_n, int* static_link) {
  return lgc::guard([&] {
    if (!ctx || !hand || !patches || !raw || !p || m < 0 || c0 < 0)
      throw std::invalid_argument("lg_place_batch: bad argument");
    if (m == 0) return;
    use_ctx(ctx);
    RunOut ro;
    PlaceOnly po;
    po.c0 = c0;
    po.m = m;
    lg_run_params q = *p;
    q.passes = 1;
    q.want_trace = 0;
    q.shard_count = 1;
    run_batch_device(ctx, *hand, *patches, field, raw, n_raw, q, ro, &po);
    std::copy(po.pose.begin(), po.pose.end(), pose);
    std::copy(po.acc.begin(), po.acc.end(), accepted);
    std::copy(po.pen.begin(), po.pen.end(), penetration);
    std::copy(po.nst.begin(), po.nst.end(), n_static);
    if (static_p) std::copy(po.stp.begin(), po.stp.end(), static_p);
    if (static_n) std::copy(po.stn.begin(), po.stn.end(), static_n);
    if (static_link) std::copy(po.stl.begin(), po.stl.end(), static_link);
  });
}

int lg_optimize_contacts_batch(lg_ctx* ctx, int m, int k, const long long* dom_off,
                               const double* dom_pos, const double* dom_nrm, const int* n_static,
                               const double* static_p, const double* static_n,
                               const lg_run_params* p, const uint64_t* seeds, int* element_ids,
                               double* objective, int* anchor, double* alpha, double* beta_x,
                               double* beta_y, long long* evaluations) {
  return lgc::guard([&] {
    if (!ctx || !p || m < 0 || (m && (!dom_off || !dom_pos || !dom_nrm || !seeds)))
      throw std::invalid_argument("lg_optimize_contacts_batch: bad argument");
    // contact_opt.cpp:49-59 (messages as the reference words them)
    if (k < 1) throw std::invalid_argument("optimize_contacts: no domains");
    if (k > kMaxK) throw std::invalid_argument("optimize_contacts: device limit is 5 domains");
    if (m == 0) return;
    for (long long t = 0; t < (long long)m * k; ++t)
      if (dom_off[t + 1] <= dom_off[t]) throw std::invalid_argument("optimize_contacts: empty domain");
    if (p->sigma <= 0.0 || p->n_inner < 1 || p->n_outer < 0 || p->restarts < 1)
      throw std::invalid_argument("optimize_contacts: bad parameters");
    use_ctx(ctx);
    cudaStream_t s = ctx->stream;
    const long long nel = dom_off[(size_t)m * k] - dom_off[0];
    std::vector<long long> eloff(dom_off, dom_off + (size_t)m * k + 1);
    for (auto& o : eloff) o -= dom_off[0];
    std::vector<int> aidx(m), nst(m, 0);
    for (int i = 0; i < m; ++i) {
      aidx[i] = i;
      nst[i] = n_static ? n_static[i] : 0;
      if (nst[i] < 0 || nst[i] > 1)
        throw std::invalid_argument("optimize_contacts: device limit is one static contact");
    }
    std::vector<double> sp(3 * (size_t)m, 0.0), sn(3 * (size_t)m, 0.0);
    if (static_p) std::copy(static_p, static_p + 3 * (size_t)m, sp.begin());
    if (static_n) std::copy(static_n, static_n + 3 * (size_t)m, sn.begin());
    const int R = p->restarts;
    const long long per_restart = k + 2ll * p->n_outer * k * p->n_inner;
    const long long per_cand = (long long)R * per_restart;
    Buf ba, bn, bsp, bsn, bo, bp, bnr, bsd, bdr, boid, bobj, ban, bsol, bbal;
    int* d_aidx = dupload(ba, aidx.data(), aidx.size(), s);
    int* d_nst = dupload(bn, nst.data(), nst.size(), s);
    double* d_stp = dupload(bsp, sp.data(), sp.size(), s);
    double* d_stn = dupload(bsn, sn.data(), sn.size(), s);
    long long* d_eloff = dupload(bo, eloff.data(), eloff.size(), s);
    double* d_elp = dupload(bp, dom_pos + 3 * dom_off[0], 3 * (size_t)nel, s);
    double* d_eln = dupload(bnr, dom_nrm + 3 * dom_off[0], 3 * (size_t)nel, s);
    uint64_t* d_seeds = dupload(bsd, seeds, (size_t)m, s);
    uint64_t* d_draws = dalloc<uint64_t>(bdr, (size_t)m * per_cand);
    lgd::k_copt_draws_seeded<<<grid_for(m, 64), 64, 0, s>>>(m, d_seeds, per_cand, d_draws);
    check_launch();
    LAUNCH(ctx);
    const int prp = p->n_outer * k * p->n_inner;
    const long long np = (long long)m * R * prp;
    if (np > 0) {
      k_copt_normals<<<grid_for(np, 256), 256, 0, s>>>(np, prp, k, per_restart, p->sigma, d_draws);
      check_launch();
      LAUNCH(ctx);
    }
    int* d_oid = dalloc<int>(boid, (size_t)m * kMaxK);
    double* d_oobj = dalloc<double>(bobj, (size_t)m);
    int* d_oan = dalloc<int>(ban, (size_t)m);
    double* d_osol = dalloc<double>(bsol, (size_t)m * 3 * kMaxC);
    int* d_bal = dalloc<int>(bbal, (size_t)m);
    CoptCfg co;
    co.k = k;
    co.n_outer = p->n_outer;
    co.n_inner = p->n_inner;
    co.restarts = R;
    co.sigma = p->sigma;
    co.lambda = p->lambda_torque;
    co.mu = p->mu;
    co.o.iterations = p->pgd_iterations;
    co.o.warm_iterations = p->pgd_warm_iterations;
    co.o.step = p->pgd_step;
    co.o.max_bt = 20;
    co.per_restart = per_restart;
    co.per_cand = per_cand;
    const int nw = std::min(R, 4);
    CK(cudaFuncSetAttribute(k_contact_opt2<3, 4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(k_contact_opt2<4, 4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(k_contact_opt2<kMaxC, 4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    auto kern = k + 1 <= 3 ? k_contact_opt2<3, 4, false>
                : k + 1 <= 4 ? k_contact_opt2<4, 4, false> : k_contact_opt2<kMaxC, 4, false>;
    size_t smem = k + 1 <= 3 ? copt2_smem<3>(k, nw)
                  : k + 1 <= 4 ? copt2_smem<4>(k, nw) : copt2_smem<kMaxC>(k, nw);
    DomIdx dom{};
    ElemSrc els{d_elp, d_eln, nullptr, DSamples{}, nullptr, nullptr, LLONG_MAX};
    kern<<<m, 32 * nw, smem, s>>>(m, d_aidx, co, d_nst, d_stp, d_stn, d_eloff, els, dom,
                                  d_draws, d_oid, d_oobj, d_oan, d_osol, kInf, d_bal);
    check_launch();
    LAUNCH(ctx);
    auto ids = ddownload(d_oid, (size_t)m * kMaxK, s);
    auto obj = ddownload(d_oobj, (size_t)m, s);
    auto an = ddownload(d_oan, (size_t)m, s);
    auto sol = ddownload(d_osol, (size_t)m * 3 * kMaxC, s);
    for (int i = 0; i < m; ++i) {
      for (int q = 0; q < k; ++q) element_ids[(size_t)i * k + q] = ids[(size_t)i * kMaxK + q];
      objective[i] = obj[i];
      anchor[i] = an[i];
      for (int c = 0; c < kMaxC; ++c) {
        if (alpha) alpha[(size_t)i * kMaxC + c] = sol[(size_t)i * 3 * kMaxC + c];
        if (beta_x) beta_x[(size_t)i * kMaxC + c] = sol[(size_t)i * 3 * kMaxC + kMaxC + c];
        if (beta_y) beta_y[(size_t)i * kMaxC + c] = sol[(size_t)i * 3 * kMaxC + 2 * kMaxC + c];
      }
      if (evaluations) evaluations[i] = (long long)R * (1 + (long long)p->n_outer * k * p->n_inner);
    }
  });
}

int lg_realized_contacts_batch(lg_ctx* ctx, const lg_hand_desc* hand, int m, const int* k,
                               const double* q, const int* links, const double* object_points,
                               double* realized_p, double* realized_n, int* realized_link,
                               double* residuals) {
  return lgc::guard([&] {
    if (!ctx || !hand || m < 0 || (m && (!k || !q || !links || !object_points)))
      throw std::invalid_argument("lg_realized_contacts_batch: bad argument");
    if (m == 0) return;
    use_ctx(ctx);
    cudaStream_t s = ctx->stream;
    bind_hand(ctx, *hand);
    std::vector<int> tl((size_t)m * kMaxK, 0);
    std::vector<double> op((size_t)m * kMaxK * 3, 0.0);
    std::vector<long long> first(m);
    long long off = 0;
    for (int i = 0; i < m; ++i) {
      if (k[i] < 1 || k[i] > kMaxK) throw std::invalid_argument("realize_grasp: 1..5 targets");
      first[i] = off;
      for (int c = 0; c < k[i]; ++c, ++off) {
        if (links[off] < 0 || links[off] >= hand->n_links)
          throw std::invalid_argument("solve_contact_ik: invalid target link");
        tl[(size_t)i * kMaxK + c] = links[off];
        for (int a = 0; a < 3; ++a) op[((size_t)i * kMaxK + c) * 3 + a] = object_points[3 * off + a];
      }
    }
    Buf bk, bq, bl, bo, brp, brn, brl, brs;
    int* d_k = dupload(bk, k, (size_t)m, s);
    double* d_q = dupload(bq, q, (size_t)m * hand->dof, s);
    int* d_l = dupload(bl, tl.data(), tl.size(), s);
    double* d_o = dupload(bo, op.data(), op.size(), s);
    double* d_rp = dalloc<double>(brp, op.size());
    double* d_rn = dalloc<double>(brn, op.size());
    int* d_rl = dalloc<int>(brl, tl.size());
    double* d_rs = dalloc<double>(brs, tl.size());
    lgd::k_realized<<<grid_for((long long)m * kMaxK, 64), 64, 0, s>>>(m, kMaxK, d_k, d_q, hand->dof, d_l,
                                                                     d_o, d_rp, d_rn, d_rl, d_rs);
    check_launch();
    LAUNCH(ctx);
    auto rp = ddownload(d_rp, op.size(), s);
    auto rn = ddownload(d_rn, op.size(), s);
    auto rl = ddownload(d_rl, tl.size(), s);
    auto rs = ddownload(d_rs, tl.size(), s);
    for (int i = 0; i < m; ++i)
      for (int c = 0; c < k[i]; ++c) {
        long long o = first[i] + c;
        size_t t = (size_t)i * kMaxK + c;
        for (int a = 0; a < 3; ++a) {
          if (realized_p) realized_p[3 * o + a] = rp[3 * t + a];
          if (realized_n) realized_n[3 * o + a] = rn[3 * t + a];
        }
        if (realized_link) realized_link[o] = rl[t];
        if (residuals) residuals[o] = rs[t];
      }
  });
}

int lg_collision_report_batch(lg_ctx* ctx, const lg_hand_desc* hand, int m, const double* q,
                              const double* poses, const double* samples, int n, double margin,
                              int cap, int* n_violations, int* link_a, int* link_b, double* depth,
                              double* max_penetration, int* pair_counts) {
  return lgc::guard([&] {
    if (!ctx || !hand || m < 0 || cap < 0 || (m && (!q || !poses || !n_violations)))
      throw std::invalid_argument("lg_collision_report_batch: bad argument");
    if (margin < 0.0) throw std::invalid_argument("broad_phase: negative margin");
    if (m == 0) return;
    use_ctx(ctx);
    cudaStream_t s = ctx->stream;
    bind_hand(ctx, *hand);
    for (int p = 0; p < hand->n_parts; ++p)
      if (hand->part_plane_off[p + 1] == hand->part_plane_off[p])
        throw std::invalid_argument("object_penetration: part has no face planes");
    std::vector<double> col((size_t)std::max(n, 1));
    Buf sc[6];
    for (int a = 0; a < 6; ++a) {
      for (int i = 0; i < n; ++i) col[i] = samples[6 * i + a];
      dupload(sc[a], col.data(), (size_t)n, s);
      CK(cudaStreamSynchronize(s));
    }
    DSamples S = make_samples(sc, n);
    const int cp = std::max(cap, 1);
    Buf bq, bp, bpl, bnv, ba, bb, bd, bm, bbp;
    double* d_q = dupload(bq, q, (size_t)m * hand->dof, s);
    double* d_p = dupload(bp, poses, 12 * (size_t)m, s);
    int* d_pl = dupload(bpl, hand->part_link, (size_t)hand->n_parts, s);
    int* d_nv = dalloc<int>(bnv, (size_t)m);
    int* d_a = dalloc<int>(ba, (size_t)m * cp);
    int* d_b = dalloc<int>(bb, (size_t)m * cp);
    double* d_d = dalloc<double>(bd, (size_t)m * cp);
    double* d_m = dalloc<double>(bm, (size_t)m);
    int* d_bp = dalloc<int>(bbp, 3 * (size_t)m);
    lgd::k_collision_report<<<grid_for(m, 32), 32, 0, s>>>(m, d_q, hand->dof, d_p, S, margin, d_pl, cp,
                                                         d_nv, d_a, d_b, d_d, d_m, d_bp);
    check_launch();
    LAUNCH(ctx);
    auto nv = ddownload(d_nv, (size_t)m, s);
    std::copy(nv.begin(), nv.end(), n_violations);
    if (link_a) {
      auto a = ddownload(d_a, (size_t)m * cp, s);
      std::copy(a.begin(), a.begin() + (size_t)m * cap, link_a);
    }
    if (link_b) {
      auto b = ddownload(d_b, (size_t)m * cp, s);
      std::copy(b.begin(), b.begin() + (size_t)m * cap, link_b);
    }
    if (depth) {
      auto d = ddownload(d_d, (size_t)m * cp, s);
      std::copy(d.begin(), d.begin() + (size_t)m * cap, depth);
    }
    if (max_penetration) {
      auto mp = ddownload(d_m, (size_t)m, s);
      std::copy(mp.begin(), mp.end(), max_penetration);
    }
    if (pair_counts) {
      auto bpv = ddownload(d_bp, 3 * (size_t)m, s);
      std::copy(bpv.begin(), bpv.end(), pair_counts);
    }
  });
}

}  // extern "C"
