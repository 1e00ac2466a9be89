// dev_fieldbuild.cuh — host orchestration of the device contact-field build
// (ContactFieldIndex::build, contact_field.cpp:306-334), the query-side
// finalisation (cell hash, dense grid, packed records) and the on-disk index
// cache in the reference's GGCF v1 format (contact_field.cpp:507-655).
// Included by lg_device.cu (single translation unit).
#pragma once

// ---------------------------------------------------------------- field
struct lg_field {
  lg_ctx* ctx = nullptr;
  DField f;
  DevPatches patches;
  Buf codebook, patch_link, patch_box_off, box_cell, box_patch, box_code_off, codes, rep_pn,
      rep_link, hash_run, run_start, run_count, cell_box, grid, rec, gop, grun, cmask, dl_rng,
      dl_codes;
  double dl_theta = NAN;  // theta the direction lists were built for
  std::vector<int> h_gop;  // dependency group per patch baked into rec
  long long n_vectors = 0, n_codes = 0;
  int n_runs = 0;
  double build_ms = 0.0;
  bool from_cache = false;
  // host export storage
  std::vector<double> x_codebook, x_rep_point, x_rep_normal;
  std::vector<int> x_patch_link, x_patch_box_off, x_rep_link;
  std::vector<long long> x_box_cell, x_box_code_off;
  std::vector<uint16_t> x_codes;
};

namespace {

template <typename K, typename V>
void radix_sort_pairs(lg_ctx* ctx, const K* kin, K* kout, const V* vin, V* vout, long long n,
                      int end_bit) {
  size_t bytes = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin, kout, vin, vout, (int)n, 0, end_bit,
                                     ctx->stream));
  void* tmp = ctx->tmp(bytes);
  CK(cub::DeviceRadixSort::SortPairs(tmp, bytes, kin, kout, vin, vout, (int)n, 0, end_bit,
                                     ctx->stream));
  LAUNCH(ctx);
}

int exclusive_scan_count(lg_ctx* ctx, const int* flags, int* ids, long long n) {
  size_t bytes = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, flags, ids, (int)n, ctx->stream));
  void* tmp = ctx->tmp(bytes);
  CK(cub::DeviceScan::ExclusiveSum(tmp, bytes, flags, ids, (int)n, ctx->stream));
  LAUNCH(ctx);
  int last_id = 0, last_flag = 0;
  CK(cudaMemcpyAsync(&last_id, ids + n - 1, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(&last_flag, flags + n - 1, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return last_id + last_flag;
}

// Query-side finalisation shared by the build and the cache load: boxes
// re-keyed by (cell, patch) into runs, cell hash, dense grid + records.
// Requires out->{box_cell, box_patch, box_code_off, patch_link} on the device
// and the cell range [cmin, cmax].
void finalize_field(lg_ctx* ctx, const lg_hand_desc& hd, const long long* cmin,
                    const long long* cmax, int P, long long n_boxes, lg_field* out) {
  cudaStream_t s = ctx->stream;
  const int bp = bits_for((unsigned long long)(P > 1 ? P - 1 : 1));
  const int bz = bits_for((unsigned long long)(cmax[2] - cmin[2]));
  const int by = bits_for((unsigned long long)(cmax[1] - cmin[1]));
  const int bx = bits_for((unsigned long long)(cmax[0] - cmin[0]));
  KeyLayout K2;
  K2.sh_patch = 0;
  K2.sh_z = bp;
  K2.sh_y = bp + bz;
  K2.sh_x = bp + bz + by;
  K2.sh_code = 0;
  K2.bits_total = bp + bz + by + bx;
  K2.base[0] = cmin[0];
  K2.base[1] = cmin[1];
  K2.base[2] = cmin[2];
  if (K2.bits_total > 64) throw std::runtime_error("index: packed cell key exceeds 64 bits");
  const long long* o_cell = out->box_cell.as<long long>();
  const int* o_bpatch = out->box_patch.as<int>();
  const long long* o_bco = out->box_code_off.as<long long>();
  Buf ck, ck2, cv, chd, crid;
  auto* d_ck = dalloc<unsigned long long>(ck, (size_t)n_boxes);
  auto* d_ck2 = dalloc<unsigned long long>(ck2, (size_t)n_boxes);
  auto* d_cv = dalloc<uint32_t>(cv, (size_t)n_boxes);
  auto* o_cellbox = dalloc<int>(out->cell_box, (size_t)n_boxes);
  k_cell_keys<<<grid_for(n_boxes, 256), 256, 0, s>>>(n_boxes, o_cell, o_bpatch, K2, d_ck, d_cv);
  LAUNCH(ctx);
  check_launch();
  radix_sort_pairs(ctx, d_ck, d_ck2, d_cv, (uint32_t*)o_cellbox, n_boxes, std::max(1, K2.bits_total));
  int* d_chd = dalloc<int>(chd, (size_t)n_boxes);
  int* d_crid = dalloc<int>(crid, (size_t)n_boxes);
  k_cell_heads<<<grid_for(n_boxes, 256), 256, 0, s>>>(n_boxes, d_ck2, K2.sh_z, d_chd);
  LAUNCH(ctx);
  check_launch();
  int n_runs = exclusive_scan_count(ctx, d_chd, d_crid, n_boxes);
  auto* o_rs = dalloc<int>(out->run_start, (size_t)n_runs);
  auto* o_rc = dalloc<int>(out->run_count, (size_t)n_runs);
  k_cell_runs<<<grid_for(n_boxes, 256), 256, 0, s>>>(n_boxes, d_chd, d_crid, o_rs, o_rc, n_runs);
  LAUNCH(ctx);
  check_launch();
  int cap = 1024;
  while (cap < 2 * n_runs) cap <<= 1;
  auto* o_hash = dalloc<int>(out->hash_run, (size_t)cap);
  CK(cudaMemsetAsync(o_hash, 0xff, (size_t)cap * sizeof(int), s));
  k_cell_hash_insert<<<grid_for(n_runs, 256), 256, 0, s>>>(n_runs, o_rs, o_cellbox, o_cell, cap - 1,
                                                             o_hash);
  LAUNCH(ctx);
  check_launch();
  // dense grid + packed run-ordered records for the query kernel
  int G = 0;
  std::vector<int> gol = groups_of(hd, &G);
  std::vector<int> plink(P);
  CK(cudaMemcpyAsync(plink.data(), out->patch_link.as<int>(), sizeof(int) * P, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  out->h_gop.resize(P);
  for (int p = 0; p < P; ++p)
    out->h_gop[p] = (plink[p] >= 0 && plink[p] < hd.n_links) ? gol[plink[p]] : -1;
  int* d_gop = dupload(out->gop, out->h_gop.data(), out->h_gop.size(), s);
  long long dx = cmax[0] - cmin[0] + 1, dy = cmax[1] - cmin[1] + 1, dz = cmax[2] - cmin[2] + 1;
  out->f.grid_ok = 0;
  if (dx > 0 && dy > 0 && dz > 0 && dx * dy * dz <= (64ll << 20)) {
    int2* g = dalloc<int2>(out->grid, (size_t)(dx * dy * dz));
    int* gr = dalloc<int>(out->grun, (size_t)(dx * dy * dz));
    CK(cudaMemsetAsync(g, 0, sizeof(int2) * (size_t)(dx * dy * dz), s));
    CK(cudaMemsetAsync(gr, 0xff, sizeof(int) * (size_t)(dx * dy * dz), s));
    k_grid_fill<<<grid_for(n_runs, 256), 256, 0, s>>>(n_runs, o_rs, o_rc, o_cellbox, o_cell, cmin[0],
                                                       cmin[1], cmin[2], (int)dy, (int)dz, g, gr);
    LAUNCH(ctx);
    check_launch();
    int4* rec = dalloc<int4>(out->rec, (size_t)n_boxes);
    k_rec_fill<<<grid_for(n_boxes, 256), 256, 0, s>>>(n_boxes, o_cellbox, o_bpatch, d_gop, o_bco, rec);
    LAUNCH(ctx);
    check_launch();
    out->f.grid_ok = 1;
    for (int a = 0; a < 3; ++a) out->f.gbase[a] = cmin[a];
    out->f.gdim[0] = (int)dx;
    out->f.gdim[1] = (int)dy;
    out->f.gdim[2] = (int)dz;
    out->f.grid = g;
    out->f.rec = rec;
    out->f.grun = gr;
    // code-major masks (sample_mask_cm) when they fit in 1 GiB
    const int C = out->f.C > 0 ? out->f.C : 0;
    out->f.cm_ok = 0;
    if (C > 0 && (size_t)n_runs * C * sizeof(uint32_t) <= (1ull << 30)) {
      uint32_t* cm = dalloc<uint32_t>(out->cmask, (size_t)n_runs * C);
      CK(cudaMemsetAsync(cm, 0, sizeof(uint32_t) * (size_t)n_runs * C, s));
      k_cmask_fill<<<grid_for(n_runs, 128), 128, 0, s>>>(n_runs, o_rs, o_rc, rec,
                                                          out->codes.as<uint16_t>(), C, cm);
      LAUNCH(ctx);
      check_launch();
      out->f.cmask = cm;
      out->f.cm_ok = 1;
    }
  }
  out->n_runs = n_runs;
  DField& f = out->f;
  f.P = P;
  f.patch_link = out->patch_link.as<int>();
  f.patch_box_off = out->patch_box_off.as<int>();
  f.B = n_boxes;
  f.box_cell = o_cell;
  f.box_patch = o_bpatch;
  f.box_code_off = o_bco;
  f.codes = out->codes.as<uint16_t>();
  f.rep_pn = out->rep_pn.as<double>();
  f.rep_link = out->rep_link.as<int>();
  f.hash_mask = cap - 1;
  f.hash_run = o_hash;
  f.run_start = o_rs;
  f.run_count = o_rc;
  f.cell_box = o_cellbox;
}

// ContactFieldIndex::build on the device (see dev_field.cuh).
void build_field_device(lg_ctx* ctx, const lg_hand_desc& hd, const lg_patches_desc& pd, int N,
                        double w, uint64_t seed, int C, lg_field* out) {
  if (pd.n_patches < 1) throw std::invalid_argument("index build: no patches");
  if (w <= 0.0 || N < 1) throw std::invalid_argument("index build: bad box width or N");
  cudaStream_t s = ctx->stream;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  bind_hand(ctx, hd);
  upload_patches(ctx, pd, out->patches);
  DevPatches& P = out->patches;
  auto cb = make_codebook(C);
  out->x_codebook = cb;
  const double* d_cb = dupload(out->codebook, cb.data(), cb.size(), s);
  CK(cudaEventRecord(e0, s));
  const int L = hd.n_links;
  const long long V = (long long)N * P.F;
  if (V > 0xffffffffll) throw std::invalid_argument("index build: too many contact vectors");
  Buf frames, cells, codes16, cmm;
  double* d_frames = dalloc<double>(frames, (size_t)N * L * 12);
  k_field_frames<<<grid_for(N, 128), 128, 0, s>>>(N, seed, d_frames);
  LAUNCH(ctx);
  check_launch();
  long long* d_cells = dalloc<long long>(cells, 3 * (size_t)V);
  uint16_t* d_codes = dalloc<uint16_t>(codes16, (size_t)V);
  long long* d_cmm = dalloc<long long>(cmm, 6);
  long long init[6] = {LLONG_MAX, LLONG_MAX, LLONG_MAX, LLONG_MIN, LLONG_MIN, LLONG_MIN};
  CK(cudaMemcpyAsync(d_cmm, init, sizeof(init), cudaMemcpyHostToDevice, s));
  size_t cb_smem = 3 * (size_t)C * sizeof(double);
  if (cb_smem > 200 * 1024) throw std::invalid_argument("index build: codebook too large for the device build");
  CK(cudaFuncSetAttribute(k_field_vectors, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cb_smem));
  // candidate-code lists for the quantizer's argmax (k_quantlist)
  constexpr int QR = 16, QL = 64;
  Buf qrng, qcodes;
  int2* d_qrng = dalloc<int2>(qrng, 6 * QR * QR);
  uint16_t* d_qcodes = dalloc<uint16_t>(qcodes, (size_t)6 * QR * QR * QL);
  k_quantlist<<<6 * QR * QR, 128, 0, s>>>(QR, QL, d_cb, C, d_qrng, d_qcodes);
  LAUNCH(ctx);
  check_launch();
  k_field_vectors<<<grid_for(V, 256), 256, cb_smem, s>>>(
      N, P.F, P.fp_link.as<int>(), P.fp_point.as<int>(), P.pts.as<double>(), P.nrm.as<double>(),
      d_frames, d_cb, C, w, QR, d_qrng, d_qcodes, d_cells, d_codes, d_cmm, d_cmm + 3);
  LAUNCH(ctx);
  check_launch();
  long long cmm_h[6];
  CK(cudaMemcpyAsync(cmm_h, d_cmm, sizeof(cmm_h), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  KeyLayout KL;
  int bc = bits_for((unsigned long long)(C - 1));
  int bz = bits_for((unsigned long long)(cmm_h[5] - cmm_h[2]));
  int by = bits_for((unsigned long long)(cmm_h[4] - cmm_h[1]));
  int bx = bits_for((unsigned long long)(cmm_h[3] - cmm_h[0]));
  int bp = bits_for((unsigned long long)(P.P - 1));
  KL.sh_code = 0;
  KL.sh_z = bc;
  KL.sh_y = bc + bz;
  KL.sh_x = bc + bz + by;
  KL.sh_patch = bc + bz + by + bx;
  KL.bits_total = KL.sh_patch + bp;
  KL.base[0] = cmm_h[0];
  KL.base[1] = cmm_h[1];
  KL.base[2] = cmm_h[2];
  if (KL.bits_total > 64) throw std::runtime_error("index build: packed field key exceeds 64 bits");
  Buf keys, keys2, vals, vals2, chead, bhead, cid, bid;
  auto* d_keys = dalloc<unsigned long long>(keys, (size_t)V);
  auto* d_keys2 = dalloc<unsigned long long>(keys2, (size_t)V);
  auto* d_vals = dalloc<uint32_t>(vals, (size_t)V);
  auto* d_vals2 = dalloc<uint32_t>(vals2, (size_t)V);
  k_field_keys<<<grid_for(V, 256), 256, 0, s>>>(V, P.F, P.fp_patch.as<int>(), d_cells, d_codes, KL,
                                                 d_keys, d_vals);
  LAUNCH(ctx);
  check_launch();
  radix_sort_pairs(ctx, d_keys, d_keys2, d_vals, d_vals2, V, std::max(1, KL.bits_total));
  int* d_ch = dalloc<int>(chead, (size_t)V);
  int* d_bh = dalloc<int>(bhead, (size_t)V);
  int* d_cid = dalloc<int>(cid, (size_t)V);
  int* d_bid = dalloc<int>(bid, (size_t)V);
  k_field_heads<<<grid_for(V, 256), 256, 0, s>>>(V, d_keys2, KL.sh_z, d_ch, d_bh);
  LAUNCH(ctx);
  check_launch();
  long long n_codes = exclusive_scan_count(ctx, d_ch, d_cid, V);
  long long n_boxes = exclusive_scan_count(ctx, d_bh, d_bid, V);
  auto* o_codes = dalloc<uint16_t>(out->codes, (size_t)n_codes);
  auto* o_rep = dalloc<double>(out->rep_pn, 6 * (size_t)n_codes);
  auto* o_rlink = dalloc<int>(out->rep_link, (size_t)n_codes);
  auto* o_cell = dalloc<long long>(out->box_cell, 3 * (size_t)n_boxes);
  auto* o_bpatch = dalloc<int>(out->box_patch, (size_t)n_boxes);
  auto* o_bco = dalloc<long long>(out->box_code_off, (size_t)n_boxes + 1);
  auto* o_pbo = dalloc<int>(out->patch_box_off, (size_t)P.P + 1);
  k_field_emit<<<grid_for(V, 256), 256, 0, s>>>(V, P.F, d_keys2, d_vals2, d_ch, d_bh, d_cid, d_bid,
                                                 d_cells, P.fp_patch.as<int>(), P.fp_point.as<int>(),
                                                 P.fp_link.as<int>(), P.pts.as<double>(),
                                                 P.nrm.as<double>(), KL, o_codes, o_rep, o_rlink,
                                                 o_cell, o_bpatch, o_bco, o_pbo);
  LAUNCH(ctx);
  check_launch();
  int nb_i = (int)n_boxes;
  long long nc_ll = n_codes;
  CK(cudaMemcpyAsync(o_pbo + P.P, &nb_i, sizeof(int), cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(o_bco + n_boxes, &nc_ll, sizeof(long long), cudaMemcpyHostToDevice, s));
  dupload(out->patch_link, P.h_link.data(), P.h_link.size(), s);
  CK(cudaStreamSynchronize(s));
  out->f.C = C;
  finalize_field(ctx, hd, cmm_h, cmm_h + 3, P.P, n_boxes, out);
  CK(cudaEventRecord(e1, s));
  CK(cudaStreamSynchronize(s));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  out->build_ms = ms;
  out->n_vectors = V;
  out->n_codes = n_codes;
  out->f.w = w;
  out->f.C = C;
  out->f.codebook = d_cb;
}

// Direction lists for the code-major query at this theta (built once per
// (field, theta) on the device).  Returns false when the path is off.
bool ensure_dirlists(lg_field* fl, double theta) {
  DField& f = fl->f;
  if (!f.grid_ok || !f.cm_ok || !(theta <= 0.99999)) return false;
  if (fl->dl_theta == theta) return true;
  constexpr int R = 32, LMAX = 96;
  cudaStream_t s = fl->ctx->stream;
  int2* rng = dalloc<int2>(fl->dl_rng, 6 * R * R);
  uint16_t* codes = dalloc<uint16_t>(fl->dl_codes, (size_t)6 * R * R * LMAX);
  k_dirlist<<<6 * R * R, 128, 0, s>>>(R, LMAX, f.codebook, f.C, theta, rng, codes);
  LAUNCH(fl->ctx);
  check_launch();
  f.dl_R = R;
  f.dl_rng = rng;
  f.dl_codes = codes;
  fl->dl_theta = theta;
  return true;
}

// Host CSR copy of a device field (lg_field_export).
void export_field(lg_field* f) {
  cudaStream_t s = f->ctx->stream;
  const DField& F = f->f;
  f->x_patch_link = ddownload(F.patch_link, (size_t)F.P, s);
  f->x_patch_box_off = ddownload(F.patch_box_off, (size_t)F.P + 1, s);
  f->x_box_cell = ddownload(F.box_cell, 3 * (size_t)F.B, s);
  f->x_box_code_off = ddownload(F.box_code_off, (size_t)F.B + 1, s);
  f->x_codes = ddownload(F.codes, (size_t)f->n_codes, s);
  f->x_rep_link = ddownload(F.rep_link, (size_t)f->n_codes, s);
  auto pn = ddownload(F.rep_pn, 6 * (size_t)f->n_codes, s);
  f->x_rep_point.resize(3 * f->n_codes);
  f->x_rep_normal.resize(3 * f->n_codes);
  for (long long c = 0; c < f->n_codes; ++c)
    for (int a = 0; a < 3; ++a) {
      f->x_rep_point[3 * c + a] = pn[6 * c + a];
      f->x_rep_normal[3 * c + a] = pn[6 * c + 3 + a];
    }
}

// --------------------------------------------------------- GGCF v1 cache
// Median-split BVHs (contact_field.cpp:182-224, bounds inflated 1e-9 at
// :22,259): part of the reference's file format, built on the host at save.
struct HAabb {
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  void expand(const HAabb& b) {
    for (int a = 0; a < 3; ++a) {
      mn[a] = b.mn[a] < mn[a] ? b.mn[a] : mn[a];
      mx[a] = b.mx[a] > mx[a] ? b.mx[a] : mx[a];
    }
  }
  void expand_pt(const double* p) {
    for (int a = 0; a < 3; ++a) {
      mn[a] = p[a] < mn[a] ? p[a] : mn[a];
      mx[a] = p[a] > mx[a] ? p[a] : mx[a];
    }
  }
  void center(double* c) const {
    for (int a = 0; a < 3; ++a) c[a] = 0.5 * (mn[a] + mx[a]);
  }
};
struct HNode {
  HAabb b;
  int32_t left = -1, right = -1, leaf = -1;
};

int32_t host_bvh(std::vector<HNode>& nodes, std::vector<std::pair<HAabb, int32_t>>& items, int lo,
                 int hi) {
  if (hi - lo == 1) {
    HNode n;
    n.b = items[lo].first;
    n.leaf = items[lo].second;
    nodes.push_back(n);
    return (int32_t)nodes.size() - 1;
  }
  HAabb cb;
  for (int i = lo; i < hi; ++i) {
    double c[3];
    items[i].first.center(c);
    cb.expand_pt(c);
  }
  double ext[3] = {cb.mx[0] - cb.mn[0], cb.mx[1] - cb.mn[1], cb.mx[2] - cb.mn[2]};
  int axis = 0;
  if (ext[1] > ext[0]) axis = 1;
  if (ext[2] > ext[axis]) axis = 2;
  std::sort(items.begin() + lo, items.begin() + hi,
            [axis](const std::pair<HAabb, int32_t>& a, const std::pair<HAabb, int32_t>& b) {
              double ca[3], cbv[3];
              a.first.center(ca);
              b.first.center(cbv);
              return ca[axis] != cbv[axis] ? ca[axis] < cbv[axis] : a.second < b.second;
            });
  int mid = lo + (hi - lo) / 2;
  int32_t l = host_bvh(nodes, items, lo, mid);
  int32_t r = host_bvh(nodes, items, mid, hi);
  HNode n;
  n.b = nodes[l].b;
  n.b.expand(nodes[r].b);
  n.left = l;
  n.right = r;
  nodes.push_back(n);
  return (int32_t)nodes.size() - 1;
}

template <typename T>
void put(std::vector<char>& o, const T& v) {
  const char* p = reinterpret_cast<const char*>(&v);
  o.insert(o.end(), p, p + sizeof(T));
}

void put_nodes(std::vector<char>& o, const std::vector<HNode>& nodes, int32_t root) {
  put(o, (uint64_t)nodes.size());
  for (const HNode& n : nodes) {
    for (int a = 0; a < 3; ++a) put(o, n.b.mn[a]);
    for (int a = 0; a < 3; ++a) put(o, n.b.mx[a]);
    put(o, n.left);
    put(o, n.right);
    put(o, n.leaf);
  }
  put(o, root);
}

// ContactFieldIndex::save (contact_field.cpp:570-600), byte for byte.
void save_field(lg_field* f, const char* path, uint64_t key) {
  export_field(f);
  const DField& F = f->f;
  const double w = F.w;
  std::vector<char> o;
  put(o, (uint32_t)0x47474346u);  // "GGCF"
  put(o, (uint32_t)1u);
  put(o, key);
  put(o, w);
  put(o, (uint32_t)F.C);
  for (double d : f->x_codebook) put(o, d);
  // the reference's index holds only patches that received a vector
  // (std::map<patch_id, ...> in insertion, :279-288), in id order
  std::vector<int> present;
  for (int p = 0; p < F.P; ++p)
    if (f->x_patch_box_off[p + 1] > f->x_patch_box_off[p]) present.push_back(p);
  put(o, (uint64_t)present.size());
  std::vector<std::pair<HAabb, int32_t>> tops;
  std::vector<HNode> top_nodes;
  for (int p : present) {
    put(o, (int32_t)p);
    put(o, (int32_t)f->x_patch_link[p]);
    int b0 = f->x_patch_box_off[p], b1 = f->x_patch_box_off[p + 1];
    put(o, (uint64_t)(b1 - b0));
    std::vector<std::pair<HAabb, int32_t>> items;
    for (int b = b0; b < b1; ++b) {
      const long long* c = &f->x_box_cell[3 * b];
      for (int a = 0; a < 3; ++a) put(o, (int64_t)c[a]);
      long long q0 = f->x_box_code_off[b], q1 = f->x_box_code_off[b + 1];
      put(o, (uint32_t)(q1 - q0));
      for (long long q = q0; q < q1; ++q) {
        put(o, f->x_codes[q]);
        put(o, (int32_t)f->x_rep_link[q]);
        for (int a = 0; a < 3; ++a) put(o, f->x_rep_point[3 * q + a]);
        for (int a = 0; a < 3; ++a) put(o, f->x_rep_normal[3 * q + a]);
      }
      HAabb cbx;  // cell_bounds(...).inflated(kBoundsEps)
      for (int a = 0; a < 3; ++a) {
        cbx.mn[a] = c[a] * w - 1e-9;
        cbx.mx[a] = (c[a] + 1) * w + 1e-9;
      }
      items.push_back({cbx, (int32_t)(b - b0)});
    }
    std::vector<HNode> nodes;
    int32_t root = host_bvh(nodes, items, 0, (int)items.size());
    put_nodes(o, nodes, root);
    tops.push_back({nodes[root].b, (int32_t)tops.size()});
  }
  int32_t top_root = -1;
  if (!tops.empty()) top_root = host_bvh(top_nodes, tops, 0, (int)tops.size());
  put_nodes(o, top_nodes, top_root);
  FILE* fp = std::fopen(path, "wb");
  if (!fp) throw std::runtime_error(std::string("cannot write index file: ") + path);
  size_t wr = std::fwrite(o.data(), 1, o.size(), fp);
  std::fclose(fp);
  if (wr != o.size()) throw std::runtime_error(std::string("short write on index file: ") + path);
}

// ContactFieldIndex::load (contact_field.cpp:602-655): false when the file
// is missing, malformed, another version, or keyed differently.
bool load_field(lg_ctx* ctx, const lg_hand_desc& hd, const char* path, uint64_t key, lg_field* out) {
  FILE* fp = std::fopen(path, "rb");
  if (!fp) return false;
  std::vector<char> buf;
  char tmp[1 << 16];
  size_t n;
  while ((n = std::fread(tmp, 1, sizeof(tmp), fp)) > 0) buf.insert(buf.end(), tmp, tmp + n);
  std::fclose(fp);
  size_t pos = 0;
  auto get = [&](auto& v) {
    if (pos + sizeof(v) > buf.size()) return false;
    std::memcpy(&v, buf.data() + pos, sizeof(v));
    pos += sizeof(v);
    return true;
  };
  uint32_t magic = 0, version = 0, cb = 0;
  uint64_t k = 0, np = 0;
  double w = 0;
  if (!get(magic) || magic != 0x47474346u) return false;
  if (!get(version) || version != 1u) return false;
  if (!get(k) || k != key) return false;
  if (!get(w) || !get(cb) || cb == 0 || cb > 65536) return false;
  std::vector<double> codebook(3 * (size_t)cb);
  for (double& d : codebook)
    if (!get(d)) return false;
  if (!get(np)) return false;
  std::vector<int> pid_of, plink;        // file order
  std::vector<long long> cells, bco{0};
  std::vector<int> bpatch;
  std::vector<uint16_t> codes;
  std::vector<int> rlink;
  std::vector<double> rpn;
  auto skip_nodes = [&]() {
    uint64_t c = 0;
    if (!get(c)) return false;
    size_t bytes = (size_t)c * (6 * sizeof(double) + 3 * sizeof(int32_t)) + sizeof(int32_t);
    if (pos + bytes > buf.size()) return false;
    pos += bytes;
    return true;
  };
  if (np == 0 || np > (1u << 24)) return false;
  for (uint64_t p = 0; p < np; ++p) {
    int32_t pid = 0, link = 0;
    uint64_t nb = 0;
    if (!get(pid) || !get(link) || !get(nb)) return false;
    // ids ascend (std::map order); the device index is keyed by id
    if (pid < 0 || (!pid_of.empty() && pid <= pid_of.back()) || pid > (1 << 24)) return false;
    pid_of.push_back(pid);
    plink.push_back(link);
    for (uint64_t b = 0; b < nb; ++b) {
      int64_t c[3];
      uint32_t ncode = 0;
      if (!get(c[0]) || !get(c[1]) || !get(c[2]) || !get(ncode)) return false;
      cells.insert(cells.end(), {c[0], c[1], c[2]});
      bpatch.push_back(pid);
      for (uint32_t q = 0; q < ncode; ++q) {
        uint16_t code = 0;
        int32_t rl = 0;
        double v[6];
        if (!get(code) || !get(rl)) return false;
        for (double& d : v)
          if (!get(d)) return false;
        if (code >= cb) return false;
        codes.push_back(code);
        rlink.push_back(rl);
        rpn.insert(rpn.end(), v, v + 6);
      }
      bco.push_back((long long)codes.size());
    }
    if (!skip_nodes()) return false;
  }
  if (!skip_nodes()) return false;
  if (cells.empty()) return false;
  cudaStream_t s = ctx->stream;
  bind_hand(ctx, hd);
  const int P = pid_of.back() + 1;
  const long long B = (long long)(cells.size() / 3);
  std::vector<int> pbo(P + 1, 0), plink_id(P, -1);
  for (size_t i = 0; i < pid_of.size(); ++i) plink_id[pid_of[i]] = plink[i];
  for (long long b = 0; b < B; ++b) ++pbo[bpatch[b] + 1];
  for (int p = 0; p < P; ++p) pbo[p + 1] += pbo[p];
  long long cmin[3] = {LLONG_MAX, LLONG_MAX, LLONG_MAX}, cmax[3] = {LLONG_MIN, LLONG_MIN, LLONG_MIN};
  for (long long b = 0; b < B; ++b)
    for (int a = 0; a < 3; ++a) {
      cmin[a] = std::min(cmin[a], cells[3 * b + a]);
      cmax[a] = std::max(cmax[a], cells[3 * b + a]);
    }
  out->x_codebook = codebook;
  const double* d_cb = dupload(out->codebook, codebook.data(), codebook.size(), s);
  dupload(out->patch_link, plink_id.data(), plink_id.size(), s);
  dupload(out->patch_box_off, pbo.data(), pbo.size(), s);
  dupload(out->box_cell, cells.data(), cells.size(), s);
  dupload(out->box_patch, bpatch.data(), bpatch.size(), s);
  dupload(out->box_code_off, bco.data(), bco.size(), s);
  dupload(out->codes, codes.data(), codes.size(), s);
  dupload(out->rep_link, rlink.data(), rlink.size(), s);
  dupload(out->rep_pn, rpn.data(), rpn.size(), s);
  CK(cudaStreamSynchronize(s));
  out->f.C = (int)cb;
  finalize_field(ctx, hd, cmin, cmax, P, B, out);
  CK(cudaStreamSynchronize(s));
  out->n_codes = (long long)codes.size();
  out->n_vectors = 0;
  out->from_cache = true;
  out->f.w = w;
  out->f.C = (int)cb;
  out->f.codebook = d_cb;
  return true;
}

}  // namespace
