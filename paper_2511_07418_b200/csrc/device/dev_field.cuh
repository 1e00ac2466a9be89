// dev_field.cuh — contact-field construction and query on the GPU.
//
// Build (reference ContactFieldIndex::build, contact_field.cpp:306-334 with
// insert_vector :279-288 and finalize_index :234-277): the std::map
// accumulation "first inserted representative per (patch, cell, code) wins,
// boxes in lexicographic cell order, codes ascending" is reproduced as a
// stable radix sort of packed (patch, cell, code) keys carrying the insertion
// index (config-major, then patch, then field point), followed by run-head
// compaction: the head of every equal-key run is its first-inserted vector.
//
// Query (query_domains :380-448): BVH traversal with closed, 1e-9-inflated
// cell bounds only ever reports the box whose cell equals floor(p / w), and
// a patch owns at most one box per cell, so a query is an exact cell lookup.
// The device index is a hash from cell to the run of boxes sharing that cell,
// sorted by patch (the reference's hit order).
#pragma once

#include <cub/cub.cuh>

#include "dev_geom.cuh"

namespace lgd {

struct DField {
  double w;
  int C;
  const double* codebook;  // [C][3]
  int P;
  const int* patch_link;     // [P]
  const int* patch_box_off;  // [P+1]
  long long B;
  const long long* box_cell;      // [B][3]
  const int* box_patch;           // [B]
  const long long* box_code_off;  // [B+1]
  const uint16_t* codes;          // [n_codes]
  const double* rep_pn;           // [n_codes][6] representative point, normal (link frame)
  const int* rep_link;            // [n_codes] representative link
  // cell hash: run r covers cell_box[run_start[r] .. run_start[r]+run_count[r])
  int hash_mask;
  const int* hash_run;  // [mask+1] run id or -1
  const int* run_start;
  const int* run_count;
  const int* cell_box;  // box ids ordered by (cell, patch)
  // dense query path (when the field's cell range is small): grid cell ->
  // (start, count) into rec; rec[j] = (dependency group of the box's patch,
  // first code, code count, box id) in (cell, patch) order.
  int grid_ok;
  long long gbase[3];
  int gdim[3];
  const int2* grid;
  const int4* rec;
  // code-major query path: grun = run id per grid cell (-1 empty);
  // cmask[run][code] = OR of group bits of the cell's boxes holding code;
  // dl_* = codes that can pass the theta test for directions in each cell
  // of a cube map over the sphere (count -1: test every code).
  const int* grun;
  const uint32_t* cmask;
  int cm_ok;
  int dl_R;
  const int2* dl_rng;
  const uint16_t* dl_codes;
};

__device__ __forceinline__ uint64_t cell_hash(long long x, long long y, long long z) {
  return mix64((uint64_t)x * 0x9E3779B97F4A7C15ull ^ (uint64_t)y * 0xC2B2AE3D27D4EB4Full ^
               (uint64_t)z * 0x165667B19E3779F9ull);
}

// cell_of (contact_field.cpp:176-180): division, not multiplication by 1/w.
__device__ __forceinline__ void cell_of(V3 p, double w, long long* c) {
  c[0] = (long long)floor(p.x / w);
  c[1] = (long long)floor(p.y / w);
  c[2] = (long long)floor(p.z / w);
}

__device__ __forceinline__ int find_run(const DField& f, const long long* c) {
  uint64_t h = cell_hash(c[0], c[1], c[2]) & (uint64_t)f.hash_mask;
  for (;;) {
    int r = f.hash_run[h];
    if (r < 0) return -1;
    int b = f.cell_box[f.run_start[r]];
    const long long* bc = f.box_cell + 3 * b;
    if (bc[0] == c[0] && bc[1] == c[1] && bc[2] == c[2]) return r;
    h = (h + 1) & (uint64_t)f.hash_mask;
  }
}

// Cube map over directions: face f in 0..5 = +x,-x,+y,-y,+z,-z, (u, v) in
// [-1, 1]^2 on the face, R x R cells.  Returns -1 for a zero / non-finite m.
__host__ __device__ __forceinline__ V3 cube_dir(int face, double u, double v) {
  switch (face) {
    case 0: return v3(1.0, u, v);
    case 1: return v3(-1.0, u, v);
    case 2: return v3(u, 1.0, v);
    case 3: return v3(u, -1.0, v);
    case 4: return v3(u, v, 1.0);
    default: return v3(u, v, -1.0);
  }
}
__device__ __forceinline__ int cube_cell(V3 m, int R) {
  double ax = fabs(m.x), ay = fabs(m.y), az = fabs(m.z);
  int face;
  double u, v, d;
  if (ax >= ay && ax >= az) {
    face = m.x > 0.0 ? 0 : 1;
    d = ax;
    u = m.y;
    v = m.z;
  } else if (ay >= az) {
    face = m.y > 0.0 ? 2 : 3;
    d = ay;
    u = m.x;
    v = m.z;
  } else {
    face = m.z > 0.0 ? 4 : 5;
    d = az;
    u = m.x;
    v = m.y;
  }
  if (!(d > 0.0) || !(d <= 1.7976931348623157e308)) return -1;
  u /= d;
  v /= d;
  double fi = (u + 1.0) * 0.5 * R, fj = (v + 1.0) * 0.5 * R;
  if (!(fi >= -1.0 && fi <= R + 1.0 && fj >= -1.0 && fj <= R + 1.0)) return -1;
  int i = (int)fi, j = (int)fj;
  i = i < 0 ? 0 : (i >= R ? R - 1 : i);
  j = j < 0 ? 0 : (j >= R ? R - 1 : j);
  return (face * R + i) * R + j;
}

// ------------------------------------------------------------ field build
// field_config (contact_field.cpp:101-114) + FK: one thread per config.
__global__ void k_field_frames(int N, uint64_t seed, double* frames) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  DRng rng;
  rng.seed(mix_seed(seed, 0x636f6e66ull, (uint64_t)c));
  double q[kMaxDof];
  for (int j = 0; j < c_hand.dof; ++j) q[j] = rng.uniform(c_hand.jlo[j], c_hand.jhi[j]);
  Xf fr[kMaxLinks];
  fk(q, fr);
  double* out = frames + (size_t)c * c_hand.n_links * 12;
  for (int l = 0; l < c_hand.n_links; ++l) {
    m3_store(out + 12 * l, fr[l].R);
    v3_store(out + 12 * l + 9, fr[l].t);
  }
}

// Contact vectors: one thread per (config, field point); quantize_normal
// (:160-172) as a 256-way argmax over a shared-memory codebook, strict '>'
// so the lowest code wins ties.
__global__ void k_field_vectors(int N, int F, const int* fp_link, const int* fp_point,
                                const double* pts, const double* nrm, const double* frames,
                                const double* codebook, int C, double w, int qR,
                                const int2* qrng, const uint16_t* qcodes, long long* cells,
                                uint16_t* codes, long long* cmin, long long* cmax) {
  extern __shared__ double s_cb[];
  for (int i = threadIdx.x; i < 3 * C; i += blockDim.x) s_cb[i] = codebook[i];
  __syncthreads();
  long long lmin[3] = {LLONG_MAX, LLONG_MAX, LLONG_MAX};
  long long lmax[3] = {LLONG_MIN, LLONG_MIN, LLONG_MIN};
  const long long V = (long long)N * F;
  for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < V;
       v += (long long)gridDim.x * blockDim.x) {
    int c = (int)(v / F);
    int f = (int)(v - (long long)c * F);
    int link = fp_link[f];
    int pi = fp_point[f];
    const double* fr = frames + ((size_t)c * c_hand.n_links + link) * 12;
    Xf x;
    x.R = m3_load(fr);
    x.t = v3_load(fr + 9);
    V3 pos = xf_apply(x, v3_load(pts + 3 * pi));
    V3 n = xf_rotate(x, v3_load(nrm + 3 * pi));
    int best = 0;
    double best_dot = -2.0;
    // the codes of n's cube-map cell (ascending; they include every code
    // that can be the argmax anywhere in the cell) or, off the fast path,
    // the whole codebook: the same first-max code either way
    double n2 = dot(n, n);
    int cell = (qR > 0 && n2 >= 1.0 - 1e-9 && n2 <= 1.0 + 1e-9) ? cube_cell(n, qR) : -1;
    int2 rg = cell >= 0 ? qrng[cell] : make_int2(0, -1);
    if (rg.y >= 0) {
      for (int t = 0; t < rg.y; ++t) {
        int i = qcodes[rg.x + t];
        double d = dot(v3(s_cb[3 * i], s_cb[3 * i + 1], s_cb[3 * i + 2]), n);
        if (d > best_dot) {
          best_dot = d;
          best = i;
        }
      }
    } else {
      for (int i = 0; i < C; ++i) {
        double d = dot(v3(s_cb[3 * i], s_cb[3 * i + 1], s_cb[3 * i + 2]), n);
        if (d > best_dot) {
          best_dot = d;
          best = i;
        }
      }
    }
    long long cl[3];
    cell_of(pos, w, cl);
    cells[3 * v] = cl[0];
    cells[3 * v + 1] = cl[1];
    cells[3 * v + 2] = cl[2];
    codes[v] = (uint16_t)best;
    for (int a = 0; a < 3; ++a) {
      lmin[a] = cl[a] < lmin[a] ? cl[a] : lmin[a];
      lmax[a] = cl[a] > lmax[a] ? cl[a] : lmax[a];
    }
  }
  for (int a = 0; a < 3; ++a) {
    for (int o = 16; o > 0; o >>= 1) {
      long long mn = __shfl_xor_sync(0xffffffffu, lmin[a], o);
      long long mx = __shfl_xor_sync(0xffffffffu, lmax[a], o);
      lmin[a] = mn < lmin[a] ? mn : lmin[a];
      lmax[a] = mx > lmax[a] ? mx : lmax[a];
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMin((long long*)&cmin[a], lmin[a]);
      atomicMax((long long*)&cmax[a], lmax[a]);
    }
  }
}

struct KeyLayout {
  int sh_code, sh_z, sh_y, sh_x, sh_patch, bits_total;
  long long base[3];
};

// Packs (patch, cell - min, code) MSB -> LSB; the vector index rides along
// as the sort value so equal keys keep insertion order.
__global__ void k_field_keys(long long V, int F, const int* fp_patch, const long long* cells,
                             const uint16_t* codes, KeyLayout L, unsigned long long* keys,
                             uint32_t* vals) {
  for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < V;
       v += (long long)gridDim.x * blockDim.x) {
    int f = (int)(v % F);
    unsigned long long k = (unsigned long long)fp_patch[f] << L.sh_patch;
    k |= (unsigned long long)(cells[3 * v] - L.base[0]) << L.sh_x;
    k |= (unsigned long long)(cells[3 * v + 1] - L.base[1]) << L.sh_y;
    k |= (unsigned long long)(cells[3 * v + 2] - L.base[2]) << L.sh_z;
    k |= (unsigned long long)codes[v] << L.sh_code;
    keys[v] = k;
    vals[v] = (uint32_t)v;
  }
}

// Run heads: code entry = new (patch, cell, code); box = new (patch, cell).
__global__ void k_field_heads(long long V, const unsigned long long* keys, int sh_z,
                              int* code_head, int* box_head) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < V;
       i += (long long)gridDim.x * blockDim.x) {
    unsigned long long k = keys[i];
    bool ch = i == 0 || keys[i - 1] != k;
    bool bh = i == 0 || (keys[i - 1] >> sh_z) != (k >> sh_z);
    code_head[i] = ch ? 1 : 0;
    box_head[i] = bh ? 1 : 0;
  }
}

__global__ void k_field_emit(long long V, int F, const unsigned long long* keys,
                             const uint32_t* vals, const int* code_head, const int* box_head,
                             const int* code_id, const int* box_id, const long long* cells,
                             const int* fp_patch, const int* fp_point, const int* fp_link,
                             const double* pts, const double* nrm, KeyLayout L,
                             uint16_t* out_codes, double* out_rep, int* out_rlink,
                             long long* box_cell,
                             int* box_patch, long long* box_code_off, int* patch_box_off) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < V;
       i += (long long)gridDim.x * blockDim.x) {
    if (!code_head[i]) continue;
    uint32_t v = vals[i];
    int f = (int)(v % (uint32_t)F);
    int ce = code_id[i];
    out_codes[ce] = (uint16_t)((keys[i] >> L.sh_code) & ((1ull << (L.sh_z - L.sh_code)) - 1ull));
    int pi = fp_point[f];
    for (int a = 0; a < 3; ++a) {
      out_rep[6 * (long long)ce + a] = pts[3 * pi + a];
      out_rep[6 * (long long)ce + 3 + a] = nrm[3 * pi + a];
    }
    out_rlink[ce] = fp_link[f];
    if (box_head[i]) {
      int b = box_id[i];
      box_cell[3 * b] = cells[3 * (long long)v];
      box_cell[3 * b + 1] = cells[3 * (long long)v + 1];
      box_cell[3 * b + 2] = cells[3 * (long long)v + 2];
      int p = fp_patch[f];
      box_patch[b] = p;
      box_code_off[b] = ce;
      bool new_patch = i == 0 || (keys[i - 1] >> L.sh_patch) != (keys[i] >> L.sh_patch);
      if (new_patch) patch_box_off[p] = b;
    }
  }
}

// Boxes re-keyed by (cell, patch) for the cell hash.
__global__ void k_cell_keys(long long B, const long long* box_cell, const int* box_patch,
                            KeyLayout L, unsigned long long* keys, uint32_t* vals) {
  for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < B;
       b += (long long)gridDim.x * blockDim.x) {
    unsigned long long k = (unsigned long long)(box_cell[3 * b] - L.base[0]) << L.sh_x;
    k |= (unsigned long long)(box_cell[3 * b + 1] - L.base[1]) << L.sh_y;
    k |= (unsigned long long)(box_cell[3 * b + 2] - L.base[2]) << L.sh_z;
    k |= (unsigned long long)box_patch[b] << L.sh_patch;
    keys[b] = k;
    vals[b] = (uint32_t)b;
  }
}

__global__ void k_cell_heads(long long B, const unsigned long long* keys, int sh_z, int* head) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < B;
       i += (long long)gridDim.x * blockDim.x)
    head[i] = (i == 0 || (keys[i - 1] >> sh_z) != (keys[i] >> sh_z)) ? 1 : 0;
}

__global__ void k_cell_runs(long long B, const int* head, const int* run_id, int* run_start,
                            int* run_count, int n_runs) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < B;
       i += (long long)gridDim.x * blockDim.x) {
    if (!head[i]) continue;
    int r = run_id[i];
    run_start[r] = (int)i;
    long long e = i + 1;
    while (e < B && !head[e]) ++e;
    run_count[r] = (int)(e - i);
  }
  (void)n_runs;
}

// Dense grid of runs + run-ordered packed box records.
__global__ void k_grid_fill(int n_runs, const int* run_start, const int* run_count,
                            const int* cell_box, const long long* box_cell, long long bx,
                            long long by, long long bz, int dy, int dz, int2* grid, int* grun) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_runs) return;
  const long long* c = box_cell + 3 * cell_box[run_start[r]];
  long long idx = ((c[0] - bx) * dy + (c[1] - by)) * dz + (c[2] - bz);
  grid[idx] = make_int2(run_start[r], run_count[r]);
  grun[idx] = r;
}

// cmask[r][code] |= bit(group) for every (box, code) of run r; static
// patches (group -1) never enter a mask.
__global__ void k_cmask_fill(int n_runs, const int* run_start, const int* run_count,
                             const int4* rec, const uint16_t* codes, int C, uint32_t* cmask) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_runs) return;
  uint32_t* row = cmask + (size_t)r * C;
  for (int j = run_start[r]; j < run_start[r] + run_count[r]; ++j) {
    int4 b = rec[j];
    if (b.x < 0) continue;
    for (int q = b.y; q < b.y + b.z; ++q) row[codes[q]] |= 1u << b.x;
  }
}

// One block per cube cell: the codes whose direction lies within
// acos(theta) + (cell angular radius) + 1e-6 rad of the cell centre — a
// superset of the codes that can pass -dot(code, n) >= theta for any unit n
// mapped to the cell.  The exact FP64 test is still applied per code.
__global__ void k_dirlist(int R, int lmax, const double* cb, int C, double theta, int2* rng,
                          uint16_t* out) {
  __shared__ int cnt;
  __shared__ double s_cos;
  __shared__ double s_c[3];
  const int cell = blockIdx.x;
  if (threadIdx.x == 0) {
    int face = cell / (R * R), i = (cell / R) % R, j = cell % R;
    double u0 = -1.0 + 2.0 * i / R, u1 = -1.0 + 2.0 * (i + 1) / R;
    double v0 = -1.0 + 2.0 * j / R, v1 = -1.0 + 2.0 * (j + 1) / R;
    V3 c = normalized(cube_dir(face, 0.5 * (u0 + u1), 0.5 * (v0 + v1)));
    double rho = 0.0;
    double us[2] = {u0, u1}, vs[2] = {v0, v1};
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) {
        double d = dot(c, normalized(cube_dir(face, us[a], vs[b])));
        rho = fmax(rho, acos(fmin(1.0, fmax(-1.0, d))));
      }
    double lim = acos(fmin(1.0, fmax(-1.0, theta))) + rho + 1e-6;
    s_cos = lim >= 3.141592653589793 ? -2.0 : cos(lim);
    s_c[0] = c.x;
    s_c[1] = c.y;
    s_c[2] = c.z;
    cnt = 0;
  }
  __syncthreads();
  for (int code = threadIdx.x; code < C; code += blockDim.x) {
    double d = cb[3 * code] * s_c[0] + cb[3 * code + 1] * s_c[1] + cb[3 * code + 2] * s_c[2];
    if (d >= s_cos) {
      int k = atomicAdd(&cnt, 1);
      if (k < lmax) out[(size_t)cell * lmax + k] = (uint16_t)code;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) rng[cell] = make_int2(cell * lmax, cnt <= lmax ? cnt : -1);
}

__global__ void k_rec_fill(long long B, const int* cell_box, const int* box_patch,
                           const int* group_of_patch, const long long* box_code_off, int4* rec) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < B;
       j += (long long)gridDim.x * blockDim.x) {
    int b = cell_box[j];
    rec[j] = make_int4(group_of_patch[box_patch[b]], (int)box_code_off[b],
                       (int)(box_code_off[b + 1] - box_code_off[b]), b);
  }
}

__global__ void k_cell_hash_insert(int n_runs, const int* run_start, const int* cell_box,
                                   const long long* box_cell, int mask, int* hash_run) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_runs) return;
  const long long* c = box_cell + 3 * cell_box[run_start[r]];
  uint64_t h = cell_hash(c[0], c[1], c[2]) & (uint64_t)mask;
  for (;;) {
    int old = atomicCAS(&hash_run[h], -1, r);
    if (old == -1) return;
    h = (h + 1) & (uint64_t)mask;
  }
}

// --------------------------------------------------------------- queries
// Does box b pass the hit test max_code(-c.n) >= theta (contact_field.cpp:
// 417-421)?  The max is >= theta iff some code is, so the scan stops at the
// first such code: the decision is identical to the full max.
__device__ __forceinline__ bool box_hit(const DField& f, const double* cb, int b, V3 n,
                                        double theta) {
  for (long long q = f.box_code_off[b]; q < f.box_code_off[b + 1]; ++q) {
    int code = f.codes[q];
    if (-dot(v3(cb[3 * code], cb[3 * code + 1], cb[3 * code + 2]), n) >= theta) return true;
  }
  return false;
}

// Hits of one transformed sample: calls visit(patch, box_global) for every
// patch whose box at cell(p) passes the code test, in patch order
// (contact_field.cpp:412-432).
template <typename Visit>
__device__ __forceinline__ void sample_hits(const DField& f, const double* cb, V3 p, V3 n,
                                            double theta, Visit&& visit) {
  long long c[3];
  cell_of(p, f.w, c);
  int r = find_run(f, c);
  if (r < 0) return;
  int s = f.run_start[r], e = s + f.run_count[r];
  for (int j = s; j < e; ++j) {
    int b = f.cell_box[j];
    if (box_hit(f, cb, b, n, theta)) visit(f.box_patch[b], b, 0.0);
  }
}

// quantize_normal candidate lists (contact_field.cpp:160-172): for cube
// cell X with centre u and angular radius r, let a = angle to the code
// nearest u.  For any unit n in X the best code is within a + r of n
// (that code is), hence within a + 2r of u: listing every code within
// a + 2r + 1e-6 rad of u (ascending) keeps every possible argmax and every
// tie.  One block per cell; lists longer than lmax fall back to the full
// scan (count -1).
__global__ void k_quantlist(int R, int lmax, const double* cb, int C, int2* rng, uint16_t* out) {
  typedef cub::BlockScan<int, 128> Scan;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ double s_u[3], s_r, s_lim;
  __shared__ double s_best[128];
  __shared__ int s_cnt;
  const int cell = blockIdx.x;
  if (threadIdx.x == 0) {
    int face = cell / (R * R), i = (cell / R) % R, j = cell % R;
    double u0 = -1.0 + 2.0 * i / R, u1 = -1.0 + 2.0 * (i + 1) / R;
    double v0 = -1.0 + 2.0 * j / R, v1 = -1.0 + 2.0 * (j + 1) / R;
    V3 c = normalized(cube_dir(face, 0.5 * (u0 + u1), 0.5 * (v0 + v1)));
    double rho = 0.0;
    double us[2] = {u0, u1}, vs[2] = {v0, v1};
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) {
        double d = dot(c, normalized(cube_dir(face, us[a], vs[b])));
        rho = fmax(rho, acos(fmin(1.0, fmax(-1.0, d))));
      }
    s_u[0] = c.x;
    s_u[1] = c.y;
    s_u[2] = c.z;
    s_r = rho;
    s_cnt = 0;
  }
  __syncthreads();
  double mx = -2.0;  // nearest code to the centre: max dot
  for (int k = threadIdx.x; k < C; k += blockDim.x) {
    double nc = sqrt(cb[3 * k] * cb[3 * k] + cb[3 * k + 1] * cb[3 * k + 1] + cb[3 * k + 2] * cb[3 * k + 2]);
    double d = (cb[3 * k] * s_u[0] + cb[3 * k + 1] * s_u[1] + cb[3 * k + 2] * s_u[2]) / nc;
    mx = fmax(mx, d);
  }
  s_best[threadIdx.x] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = -2.0;
    for (int t = 0; t < (int)blockDim.x; ++t) m = fmax(m, s_best[t]);
    double a = acos(fmin(1.0, fmax(-1.0, m)));
    double lim = a + 2.0 * s_r + 1e-6;
    s_lim = lim >= 3.141592653589793 ? -2.0 : cos(lim);
  }
  __syncthreads();
  for (int base = 0; base < C; base += blockDim.x) {
    int k = base + threadIdx.x;
    int in = 0;
    if (k < C) {
      double nc = sqrt(cb[3 * k] * cb[3 * k] + cb[3 * k + 1] * cb[3 * k + 1] + cb[3 * k + 2] * cb[3 * k + 2]);
      double d = (cb[3 * k] * s_u[0] + cb[3 * k + 1] * s_u[1] + cb[3 * k + 2] * s_u[2]) / nc;
      in = d >= s_lim ? 1 : 0;
    }
    int pos, tot;
    Scan(tmp).ExclusiveSum(in, pos, tot);
    if (in && s_cnt + pos < lmax) out[(size_t)cell * lmax + s_cnt + pos] = (uint16_t)k;
    __syncthreads();
    if (threadIdx.x == 0) s_cnt += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) rng[cell] = make_int2(cell * lmax, s_cnt <= lmax ? s_cnt : -1);
}

// Code-major reachability mask: bit g set iff some code c passes
// -dot(c, n) >= theta and some group-g box of the cell holds c — the same
// predicate as sample_mask with the two existentials swapped.  Only codes
// of n's cube-map cell are tested (exact test; cell lists are supersets).
__device__ __forceinline__ uint32_t sample_mask_cm(const DField& f, const double* cb, V3 p, V3 n,
                                                   double theta) {
  long long c[3];
  cell_of(p, f.w, c);
  long long x = c[0] - f.gbase[0], y = c[1] - f.gbase[1], z = c[2] - f.gbase[2];
  if (x < 0 || y < 0 || z < 0 || x >= f.gdim[0] || y >= f.gdim[1] || z >= f.gdim[2]) return 0u;
  int r = f.grun[(x * f.gdim[1] + y) * f.gdim[2] + z];
  if (r < 0) return 0u;
  const uint32_t* row = f.cmask + (size_t)r * f.C;
  double n2 = dot(n, n);
  int cell = (n2 >= 1.0 - 1e-9 && n2 <= 1.0 + 1e-9) ? cube_cell(neg(n), f.dl_R) : -1;
  int2 rg = cell >= 0 ? f.dl_rng[cell] : make_int2(0, -1);
  uint32_t bits = 0u;
  if (rg.y >= 0) {
    // four listed codes at a time: the tests, then the passing codes' mask
    // words as independent loads, then the OR (an order-free reduction)
    for (int t0 = 0; t0 < rg.y; t0 += 4) {
      uint32_t w[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int code = t0 + u < rg.y ? f.dl_codes[rg.x + t0 + u] : 0;
        const bool pass = t0 + u < rg.y &&
                          -dot(v3(cb[3 * code], cb[3 * code + 1], cb[3 * code + 2]), n) >= theta;
        w[u] = pass ? row[code] : 0u;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) bits |= w[u];
    }
  } else {
    for (int code = 0; code < f.C; ++code)
      if (-dot(v3(cb[3 * code], cb[3 * code + 1], cb[3 * code + 2]), n) >= theta) bits |= row[code];
  }
  return bits;
}

// Reachability mask of one transformed sample: bit g set iff some patch of
// dependency group g has a hit box.  Boxes of static patches and of groups
// already in the mask cannot change it and are skipped.
__device__ __forceinline__ uint32_t sample_mask(const DField& f, const double* cb,
                                                const int* group_of_patch, V3 p, V3 n,
                                                double theta) {
  long long c[3];
  cell_of(p, f.w, c);
  if (f.grid_ok) {
    long long x = c[0] - f.gbase[0], y = c[1] - f.gbase[1], z = c[2] - f.gbase[2];
    if (x < 0 || y < 0 || z < 0 || x >= f.gdim[0] || y >= f.gdim[1] || z >= f.gdim[2]) return 0u;
    int2 se = f.grid[(x * f.gdim[1] + y) * f.gdim[2] + z];
    uint32_t bits = 0u;
    for (int j = se.x; j < se.x + se.y; ++j) {
      int4 r = f.rec[j];
      if (r.x < 0 || ((bits >> r.x) & 1u)) continue;
      for (int q = r.y; q < r.y + r.z; ++q) {
        int code = f.codes[q];
        if (-dot(v3(cb[3 * code], cb[3 * code + 1], cb[3 * code + 2]), n) >= theta) {
          bits |= 1u << r.x;
          break;
        }
      }
    }
    return bits;
  }
  int r = find_run(f, c);
  if (r < 0) return 0u;
  uint32_t bits = 0u;
  int s = f.run_start[r], e = s + f.run_count[r];
  for (int j = s; j < e; ++j) {
    int b = f.cell_box[j];
    int g = group_of_patch[f.box_patch[b]];
    if (g < 0 || ((bits >> g) & 1u)) continue;
    if (box_hit(f, cb, b, n, theta)) bits |= 1u << g;
  }
  return bits;
}

}  // namespace lgd
