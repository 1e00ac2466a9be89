/*
 * lg.h — C-ABI drop-in boundary of the B200-native Lightning Grasp forward pass.
 *
 * Everything on the hot path (reference proj/src/pipeline.cpp:308-625 and the
 * L2-L5 modules it calls) runs on the GPU behind lg_run_batch, lg_field_build
 * and the stage-level batch entry points below.  What the reference keeps on
 * the caller side (load_hand, load_mesh, sample_surface, decompose_patches,
 * parse_config, write_dataset — SURVEY.md 8(b)) stays with the caller, which
 * hands flat, caller-owned SoA views across: lg_hand_desc, lg_visual_desc,
 * lg_patches_desc, sample arrays and lg_run_params.  This library exports no
 * loader of its own (the repository's stand-in caller is caller/, outside the
 * product).
 *
 * Conventions:
 *   - every entry point returns an int status: LG_OK or a negative code that
 *     names the reference exception class it replaces; the message is kept in
 *     a thread-local buffer readable with lg_last_error();
 *   - handles are library-owned and freed with the matching *_destroy;
 *   - input arrays are caller-owned and copied in; output arrays are either
 *     library-owned (valid until the owning handle is destroyed) or caller
 *     buffers with an explicit capacity;
 *   - one in-flight call per lg_ctx, and one in-flight device call per GPU:
 *     the hand description is bound to the device's constant bank for the
 *     call (one context per GPU, as the multi-GPU driver uses them);
 *   - there is no CPU fallback: on a machine without a CUDA device every
 *     device entry point returns LG_ERR_CUDA.
 *
 * Arrays of 3-vectors are row-major [n][3]; rotations are row-major 3x3;
 * object samples are [n][6] = (position xyz, unit outward normal xyz).
 */
#ifndef LG_H_
#define LG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (reference exception classes) ---------- */
#define LG_OK 0
#define LG_ERR_INVALID_ARGUMENT (-1) /* std::invalid_argument */
#define LG_ERR_RUNTIME (-2)          /* std::runtime_error (I/O, config)   */
#define LG_ERR_OUT_OF_RANGE (-3)     /* std::out_of_range (reverse_lookup) */
#define LG_ERR_CUDA (-4)             /* no device / CUDA runtime failure   */
#define LG_ERR_NOMEM (-5)

#define LG_MAX_K 5          /* k_contacts range [2,5] (config.cpp:107-112) */
#define LG_MAX_CONTACTS 6   /* k slots + at most one static contact       */
#define LG_MAX_DOF 32       /* joint slots in the result records           */
#define LG_MAX_GROUPS 32    /* reachability mask is one uint32 per sample */
/* Hands the device accepts (larger ones return LG_ERR_INVALID_ARGUMENT): */
#define LG_DEVICE_MAX_DOF 24    /* actuated joints                        */
#define LG_DEVICE_MAX_LINKS 32  /* links                                  */
#define LG_DEVICE_MAX_PARTS 63  /* convex collision parts                 */
#define LG_DEVICE_MAX_CHAIN 10  /* links on a root -> link chain          */

/* Copies the calling thread's last error message; returns its length. */
int lg_last_error(char* buf, size_t cap);
/* Library build string (arch, compile flags). */
const char* lg_version(void);

/* ---- flat model descriptions (pointer views, no ownership) -------------- */

/* HandModel (reference hand.hpp:19-46).  Links are in file order; joint
 * types: 0 fixed, 1 revolute, 2 prismatic. Parts are grouped by link in link
 * order (part_link is non-decreasing). */
typedef struct lg_hand_desc {
  int n_links;
  int dof; /* actuated_count */
  int root;
  const int* parent;      /* [n_links], -1 for root */
  const int* joint_type;  /* [n_links] */
  const int* joint_index; /* [n_links], -1 when not actuated */
  const int* topo_order;  /* [n_links], parents before children */
  const double* origin_R; /* [n_links][9] parent -> pre-motion frame */
  const double* origin_t; /* [n_links][3] */
  const double* axis;     /* [n_links][3] unit, link frame */
  const double* limit_lo; /* [n_links] */
  const double* limit_hi; /* [n_links] */
  int n_parts;
  const int* part_link;      /* [n_parts] */
  const int* part_vert_off;  /* [n_parts+1] */
  const double* part_verts;  /* [*][3] link-local hull vertices */
  const int* part_tri_off;   /* [n_parts+1] */
  const int* part_tris;      /* [*][3] indices local to the part */
  const int* part_plane_off; /* [n_parts+1] */
  const double* part_planes; /* [*][4] (unit outward normal, offset) */
  const double* part_bounds; /* [n_parts][6] (min xyz, max xyz) */
} lg_hand_desc;

/* Visual meshes of the links (HandModel Link::visual, hand.hpp:27), link-local,
 * CSR over links: the input of the hand's surface sampling (pipeline.cpp:277-285). */
typedef struct lg_visual_desc {
  int n_links;
  const int* vert_off;  /* [n_links+1] */
  const double* verts;  /* [*][3] */
  const int* tri_off;   /* [n_links+1] */
  const int* tris;      /* [*][3] vertex indices local to the link */
} lg_visual_desc;

/* ContactPatch list (reference contact_field.hpp:20-30); ids are dense. */
typedef struct lg_patches_desc {
  int n_patches;
  const int* link;        /* [P] */
  const int* point_off;   /* [P+1] into points/normals */
  const double* points;   /* [*][3] link-local member samples */
  const double* normals;  /* [*][3] */
  const int* fp_off;      /* [P+1] into field_points */
  const int* field_points;/* [*] member index within the patch, sorted */
} lg_patches_desc;

/* Exported contact-field index (ContactFieldIndex, contact_field.hpp:112-137)
 * as CSR.  Box order inside a patch is lexicographic by cell (std::map order
 * of contact_field.cpp:226-227) so a box id is its rank inside its patch. */
typedef struct lg_field_csr {
  double box_width;
  int codebook_size;
  const double* codebook;   /* [C][3] */
  int n_patches;
  const int* patch_link;    /* [P] */
  const int* patch_box_off; /* [P+1] */
  long long n_boxes;
  const long long* box_cell;/* [B][3] */
  const long long* box_code_off; /* [B+1] */
  long long n_codes;
  const uint16_t* codes;    /* [n_codes] ascending within a box */
  const int* rep_link;      /* [n_codes] IndexRep.link */
  const double* rep_point;  /* [n_codes][3] IndexRep.point (link-local) */
  const double* rep_normal; /* [n_codes][3] */
  long long n_vectors;      /* swept contact vectors inserted */
} lg_field_csr;

/* RunConfig (reference config.hpp:15-77), numeric part plus asset paths. */
typedef struct lg_run_params {
  char hand[512];
  char object[512];
  char out[512];
  uint64_t seed;
  int batch, workers, passes, cache, export_obj, k_contacts;
  double samples_per_cm2, object_scale, probe_half_width, probe_depth_threshold;
  double hand_scale;
  int field_configs;
  double box_width, patch_radius;
  int field_points_per_patch, codebook_size;
  double theta_hit;
  int placement_mode; /* 0 exhaustive, 1 canonical */
  double static_contact_prob;
  double canonical_center[3], canonical_half_extents[3];
  double penetration_margin;
  double lambda_torque, mu, eps_stable;
  int pgd_iterations, pgd_warm_iterations;
  double pgd_step;
  int n_outer, n_inner, restarts;
  double sigma;
  double beta;
  int ik_iterations;
  double step_clamp, residual_tol, damping_scale;
  int finetune_rounds, finetune_iterations, lookup_attempts, unused_attempts;
  double contact_tol;
  /* B200 extensions: seed sharding (rank r of R owns c in [rB/R,(r+1)B/R)) */
  int shard_rank, shard_count;
  int want_trace; /* fill one lg_trace per (pass, candidate) */
} lg_run_params;


/* ---- results ----------------------------------------------------------- */

/* Grasp (pipeline.hpp:19-38) plus its candidate id g = pass*batch + c. */
typedef struct lg_grasp {
  long long g;
  double pose_R[9];
  double pose_t[3];
  int dof;
  double q[LG_MAX_DOF];
  int n_contacts;
  double contact_p[LG_MAX_CONTACTS][3];
  double contact_n[LG_MAX_CONTACTS][3];
  int contact_link[LG_MAX_CONTACTS];
  double objective;
  int penetration_free, stable, ik_converged;
} lg_grasp;

/* StageProfile (pipeline.hpp:44-60). Stage seconds are device time. */
typedef struct lg_profile {
  double placement_domains, contact_optimization, kinematics_optimization,
      postprocessing, total, field_build;
  long long candidates, placements_accepted, contact_sets_balanced, ik_finite,
      penetration_free, ik_converged, stable, valid;
  double grasps_per_second;
  long long patches, boxes, field_vectors, object_samples, field_samples;
  long long gpu_launches;
  /* B200 extensions: device time of the pass (CUDA events on the library
   * stream, first kernel to last kernel; input upload and result download
   * excluded), bytes moved across PCIe, and algorithmic work counters. */
  double device_seconds;
  long long h2d_bytes, d2h_bytes;
  long long ik_iterations, fk_evals, wrench_evals, wrench_grads, proj_evals;
  long long realize_calls, collision_calls;
  double realize_seconds, contact_opt_seconds;
  long long index_from_cache; /* RunResult.index.from_cache */
  long long index_codes;      /* codes (= representatives) over all boxes */
} lg_profile;

/* Per-candidate record of every stage decision, used by the stage parity
 * harness (the oracle fills the same struct). */
typedef struct lg_trace {
  long long g;
  int pass, c;
  /* stage 1: place_object + query_domains + group pick (pipeline.cpp:396-438) */
  int accepted;
  double penetration;
  double pose_R[9], pose_t[3];
  int n_static, static_link;
  double static_p[3], static_n[3];
  int n_groups;
  int domain_size[LG_MAX_GROUPS];
  int picked;
  int chosen[LG_MAX_K];
  /* stage 2: optimize_contacts + balance gate (pipeline.cpp:444-458) */
  int opt_element[LG_MAX_K];
  int opt_sample[LG_MAX_K];
  double opt_objective;
  int opt_anchor, opt_evaluations;
  double opt_alpha[LG_MAX_CONTACTS], opt_bx[LG_MAX_CONTACTS],
      opt_by[LG_MAX_CONTACTS];
  int balanced;
  /* stage 3: lookup attempts (pipeline.cpp:465-523) */
  int realized, attempts_run, best_attempt, best_clear;
  double max_residual;
  double real_q[LG_MAX_DOF];
  unsigned long long used_joints;
  int target_link[LG_MAX_K];
  double target_point[LG_MAX_K][3], target_normal[LG_MAX_K][3];
  /* stage 4: postprocess (pipeline.cpp:528-604) */
  int unused_attempt, penetration_free, ik_converged, stable, valid, dropped;
  double final_q[LG_MAX_DOF];
  double objective;
} lg_trace;

typedef struct lg_result lg_result;
int lg_result_profile(const lg_result* r, lg_profile* out);
long long lg_result_num_grasps(const lg_result* r);
const lg_grasp* lg_result_grasps(const lg_result* r);
long long lg_result_num_traces(const lg_result* r);
const lg_trace* lg_result_traces(const lg_result* r);
void lg_result_destroy(lg_result* r);

typedef struct lg_ctx lg_ctx;
typedef struct lg_patches lg_patches;

/* splitmix mix_seed (rng.hpp:25-28), the per-stream seed of every draw. */
uint64_t lg_mix_seed(uint64_t seed, uint64_t a, uint64_t b);

/* ---- device side (sm_100a) ---------------------------------------------- */

typedef struct lg_field lg_field;

int lg_device_count(int* n);
int lg_ctx_create(int device, lg_ctx** out);
void lg_ctx_destroy(lg_ctx* ctx);

/* build_field's hand steps (pipeline.cpp:277-285) on the GPU: per-link
 * sample_surface with stream 'hnds' (mesh.cpp:297-339), decompose_patches'
 * greedy cover and field-point subsets (contact_field.cpp:26-99).  Output is
 * identical to the reference's patches; read it with lg_patches_export. */
int lg_hand_patches_device(lg_ctx* ctx, const lg_hand_desc* hand, const lg_visual_desc* visual,
                           double samples_per_cm2, double patch_radius, uint64_t seed,
                           int field_cap, lg_patches** out);
int lg_patches_export(const lg_patches* p, lg_patches_desc* out);
void lg_patches_destroy(lg_patches* p);

/* ContactFieldIndex::build (contact_field.cpp:306-334) on the GPU. */
int lg_field_build(lg_ctx* ctx, const lg_hand_desc* hand,
                   const lg_patches_desc* patches, int N, double box_width,
                   uint64_t seed, int codebook_size, lg_field** out);
/* Copies the index to host CSR (pointers valid until lg_field_destroy). */
int lg_field_export(lg_field* f, lg_field_csr* out);
void lg_field_destroy(lg_field* f);
/* ContactFieldIndex::save / load (contact_field.cpp:570-655): the GGCF v1
 * file, byte-identical to the reference's. load sets *out = NULL (and returns
 * LG_OK) when the file is missing, malformed, or keyed differently — the
 * reference's std::nullopt. */
int lg_field_save(lg_field* f, const char* path, uint64_t key);
/* index_cache_key (config.cpp:403-417): the cache key of params (FNV-1a of
 * the hand file named by params->hand and the index-shaping parameters). */
int lg_index_cache_key(const lg_run_params* params, uint64_t* key);
int lg_field_load(lg_ctx* ctx, const lg_hand_desc* hand, const char* path,
                  uint64_t key, lg_field** out);

/* query_domains (contact_field.cpp:380-448) for m poses at once: writes the
 * reachability mask masks[m][n] (bit g set iff sample i is an element of group
 * g's domain) and, when scores != NULL, the element score per (pose, sample)
 * (max over all groups' hits, 0 when none). poses are [m][12] = (R row-major,
 * t). group_of_patch maps patch id -> dependency group (-1 static). */
int lg_query_domains_batch(lg_ctx* ctx, lg_field* f, const int* group_of_patch,
                           const double* samples, int n, const double* poses,
                           int m, double theta_hit, uint32_t* masks,
                           double* scores);

/* query_domains (contact_field.cpp:380-448; contact_field.hpp:98-109,147-150)
 * for ONE pose (R row-major, t): the ContactDomain of every dependency group
 * 0..n_groups-1 (group_of_patch maps patch id -> group, -1 static).  Elements
 * are in sample order within a group; each carries its sample index, posed
 * position and normal, score (max(0, best -code.n over its hits)) and its
 * hits (patch id, box id within the patch) sorted by patch.  Read with
 * lg_domains_group / lg_domains_elements; the arrays stay valid until
 * lg_domains_destroy. */
typedef struct lg_domains lg_domains;
int lg_query_domains_elements(lg_ctx* ctx, lg_field* f, const int* group_of_patch, int n_groups,
                              const double* samples, int n, const double* pose, double theta_hit,
                              lg_domains** out);
/* elements [*first, *first + *count) belong to group `group` */
int lg_domains_group(const lg_domains* d, int group, long long* first, long long* count);
/* all elements of all groups: hits of element e are [hit_off[e], hit_off[e+1]) */
int lg_domains_elements(const lg_domains* d, long long* n_elements, const int** sample,
                        const double** pos, const double** nrm, const double** score,
                        const long long** hit_off, const int** hit_patch, const int** hit_box);
void lg_domains_destroy(lg_domains* d);

/* reverse_lookup (contact_field.cpp:450-484; contact_field.hpp:154-156) for m
 * domain elements: element t has hits [hit_off[t], hit_off[t+1]) (patch id,
 * box id) and outward normal normals[t]; seeds[t] is its choice seed.
 * Writes the IndexRep: link, link-local point and normal.  An element without
 * hits or with a box outside the index returns LG_ERR_OUT_OF_RANGE, as the
 * reference throws std::out_of_range. */
int lg_reverse_lookup_batch(lg_ctx* ctx, lg_field* f, int m, const long long* hit_off,
                            const int* hit_patch, const int* hit_box, const double* normals,
                            const uint64_t* seeds, int* link, double* point, double* normal);

/* place_object (pipeline.cpp:122-183; pipeline.hpp:103-106) for candidates
 * c in [c0, c0+m): stream mix_seed(params->seed, 'plac', c), statics from
 * collect_static_surface, verdict against the preprocessed raw samples.
 * Writes pose [m][12] (R row-major, t), accepted, penetration and the static
 * contact (n_static[m] in {0,1}; static_p/n [m][3], static_link [m]).  field
 * may be NULL (built from params). */
int lg_place_batch(lg_ctx* ctx, const lg_hand_desc* hand, const lg_patches_desc* patches,
                   lg_field* field, const double* raw, int n_raw, const lg_run_params* params,
                   int c0, int m, double* pose, int* accepted, double* penetration,
                   int* n_static, double* static_p, double* static_n, int* static_link);

/* optimize_contacts (contact_opt.cpp:45-142; contact_opt.hpp:49-52) for m
 * problems of k domains each: domain (i, q) is elements
 * [dom_off[i*k+q], dom_off[i*k+q+1]) of dom_pos / dom_nrm (element positions
 * and outward normals, [*][3]); n_static[i] in {0,1} static contacts
 * (static_p / static_n [m][3], normal = inward force direction); params gives
 * n_outer, n_inner, restarts, sigma, lambda_torque, mu and the PGD settings;
 * seeds[i] the problem's stream seed.  Writes element_ids [m][k], the
 * objective, the solution (anchor; alpha / beta_x / beta_y [m][6] over
 * [slot contacts..., static]) and the number of wrench solves. */
int lg_optimize_contacts_batch(lg_ctx* ctx, int m, int k, const long long* dom_off,
                               const double* dom_pos, const double* dom_nrm, const int* n_static,
                               const double* static_p, const double* static_n,
                               const lg_run_params* params, const uint64_t* seeds,
                               int* element_ids, double* objective, int* anchor, double* alpha,
                               double* beta_x, double* beta_y, long long* evaluations);

/* realize_grasp's final projection (pipeline.cpp:196-221,250; RealizeResult
 * pipeline.hpp:108-115): for configuration q[i] and problem i's k[i] targets
 * (link, world object point; CSR like lg_realize_batch), the realized contact
 * on the hand surface (world position, outward normal, link) and the
 * position residual per target. */
int lg_realized_contacts_batch(lg_ctx* ctx, const lg_hand_desc* hand, int m, const int* k,
                               const double* q, const int* links, const double* object_points,
                               double* realized_p, double* realized_n, int* realized_link,
                               double* residuals);

/* validate_grasp_collisions' full CollisionReport (collision.cpp:230-288;
 * collision.hpp:57-65) for m configurations: violations deduplicated per
 * link pair in the reference's pair order (link_b = -1: the object; depth 0
 * for hand-hand), up to cap per configuration ([m][cap]); n_violations[i]
 * is the full count; max_penetration; pair_counts [m][3] = broad_pairs,
 * narrow_gjk, narrow_halfplane. */
int lg_collision_report_batch(lg_ctx* ctx, const lg_hand_desc* hand, int m, const double* q,
                              const double* poses, const double* samples, int n, double margin,
                              int cap, int* n_violations, int* link_a, int* link_b, double* depth,
                              double* max_penetration, int* pair_counts);

/* preprocess_object (pipeline.cpp:71-98): keep[i] = 1 when sample i survives. */
int lg_preprocess(lg_ctx* ctx, const double* samples, int n,
                  double probe_half_width, double depth_threshold,
                  uint8_t* keep);

/* Batched wrench solves (solve_fswo / solve_gswo, wrench.cpp:179-228,247-258): problem i has n[i] <= 6
 * contacts given as points/inward normals [i][6][3]; tangent frames come from
 * tangent_basis.  mode 0 = solve_fswo, 1 = solve_gswo. Outputs objective,
 * anchor, alpha/beta_x/beta_y [i][6]. */
int lg_wrench_solve_batch(lg_ctx* ctx, int m, const int* n, const double* points,
                          const double* normals, double lambda_torque, double mu,
                          int mode, int iterations, int warm_iterations,
                          double step, int max_backtracks, double* objective,
                          int* anchor, double* alpha, double* beta_x,
                          double* beta_y);

/* solve_fswo / solve_gswo (wrench.cpp:179-228,247-258) on explicit
 * WrenchProblems (wrench.hpp:14-27): problem t has n[t] <= 6 contacts with
 * points, inward normals and the caller's tangent frames [t][6][3], its own
 * lambda_torque[t] and mu[t]; mode 0 = solve_fswo, 1 = solve_gswo.  use_warm
 * (may be NULL) selects a warm start per problem from warm_alpha / beta_x /
 * beta_y [t][6] — the reference's `warm && warm->valid() && size == n` test
 * (and zero betas when the warm betas are missing) is the caller's.  Outputs
 * as lg_wrench_solve_batch. */
int lg_wrench_problem_batch(lg_ctx* ctx, int m, const int* n, const double* points,
                            const double* normals, const double* tangent_x,
                            const double* tangent_y, const double* lambda_torque,
                            const double* mu, int mode, int iterations, int warm_iterations,
                            double step, int max_backtracks, const int* use_warm,
                            const double* warm_alpha, const double* warm_beta_x,
                            const double* warm_beta_y, double* objective, int* anchor,
                            double* alpha, double* beta_x, double* beta_y);

/* Batched validate_grasp_collisions (collision.cpp:230-288): clean[i] for
 * configuration q[i] (dof) and object pose[i] (12) against the samples. */
int lg_collision_batch(lg_ctx* ctx, const lg_hand_desc* hand, int m,
                       const double* q, const double* poses,
                       const double* samples, int n, double margin,
                       uint8_t* clean, double* max_penetration);

/* Batched realize_grasp (pipeline.cpp:185-253): problem i has k[i] targets
 * (object point, inward normal, link, hand local point, hand local normal).
 * Writes q[i][dof], max residual, finite flag and used-joint bitmask. */
int lg_realize_batch(lg_ctx* ctx, const lg_hand_desc* hand, int m, const int* k,
                     const double* object_points, const double* object_normals,
                     const int* links, const double* hand_points,
                     const double* hand_normals, double beta, int iterations,
                     double step_clamp, double residual_tol,
                     double damping_scale, int finetune_rounds,
                     int finetune_iterations, double* q, double* max_residual,
                     int* finite, unsigned long long* used_joints);

/* solve_contact_ik (ik.cpp:30-139; ik.hpp:49-51) for m problems: problem i
 * has k[i] <= LG_MAX_K targets (CSR over the target arrays, as in
 * lg_realize_batch) and starts from q0 [m][dof]; the remaining arguments are
 * IkParams.  Writes q [m][dof], finite, used_joints (bit j = joint j),
 * IkResult.iterations and .objective, and per target (CSR) the position
 * residual and the cosine std::clamp(hand normal . object normal, -1, 1)
 * whose std::acos is IkResult.residuals[].normal_angle (the caller applies
 * its libm).  Invalid arguments return LG_ERR_INVALID_ARGUMENT with the
 * reference's messages. */
int lg_contact_ik_batch(lg_ctx* ctx, const lg_hand_desc* hand, int m, const int* k,
                        const double* q0, const double* object_points,
                        const double* object_normals, const int* links,
                        const double* hand_points, const double* hand_normals,
                        double beta, int iterations, double step_clamp,
                        double residual_tol, double damping_scale, double damping_min,
                        int max_backtracks, double* q, int* finite,
                        unsigned long long* used_joints, int* iterations_out,
                        double* objective, double* position_residual,
                        double* normal_cosine);

/* validate_dataset (validate.cpp:56-175) per grasp: every measured quantity
 * the reference's checks read, in its check order.  status: 0 fully checked,
 * 1 joint vector size mismatch, 2 pose not rigid, 3 joint limits violated,
 * 4 no contacts (the reference's `continue` cases).  contact_state: 0 checked,
 * 1 invalid link id, 2 normal not unit length.  wrench_error: 0 solved,
 * 1 zero normal, 2 normal not unit length (tangent_basis throws). */
typedef struct lg_grasp_check {
  int status;
  double rigid_error;
  int n_limit;
  int limit_link[LG_MAX_DOF];
  double limit_value[LG_MAX_DOF];
  int n_contacts;
  int contact_state[LG_MAX_CONTACTS];
  double hand_dist[LG_MAX_CONTACTS];
  double object_dist[LG_MAX_CONTACTS];
  double worst_depth;
  int wrench_error;
  double wrench_objective;
} lg_grasp_check;

/* validate_dataset on the GPU: n grasps against the hand, the object mesh
 * (verts [nv][3], tris [nt][3]) and its surface samples ([ns][6], the
 * sample_surface stream 'objs' the reference re-draws); p supplies
 * contact_tol, penetration_margin, lambda_torque, mu, eps_stable and the PGD
 * settings. */
int lg_validate_batch(lg_ctx* ctx, const lg_hand_desc* hand, const lg_grasp* grasps,
                      long long n, const double* obj_verts, int nv, const int* obj_tris,
                      int nt, const double* samples, int ns, const lg_run_params* p,
                      lg_grasp_check* out);
/* The reference's ValidationReport issues for these checks, one
 * "<grasp>\t<message>\n" line each, message text as validate.cpp words it.
 * Writes at most cap bytes (NUL-terminated) and the required size to
 * *needed; *n_issues receives the issue count. */
int lg_validation_issues(const char* const* joint_names, int n_links,
                         const lg_grasp_check* checks, long long n,
                         const lg_run_params* p, char* buf, size_t cap, size_t* needed,
                         long long* n_issues);

/* The hot path's transcendentals on the device (which: 0 sin, 1 cos, 2 log,
 * 3 atan2(x, y), 4 hypot(x, y)): glibc 2.39's algorithms restated in
 * csrc/lg_libm.h, used by every kernel that draws Box-Muller normals, builds a
 * rotation or projects a friction disc (rng.hpp:47-76, hand.cpp:286-288,
 * geometry.hpp:129-143, wrench.cpp:96).  Exposed for the bit-exactness check
 * against the host's std:: functions. */
int lg_libm_eval(lg_ctx* ctx, int which, long long n, const double* x, const double* y,
                 double* out);
/* With LG_CHECK_CANARY=1 in the environment every device buffer carries a
 * guard band checked at release: the number of buffers found overwritten
 * past their end so far (0 expected). */
long long lg_debug_canary_violations(void);

/* run_batch (pipeline.cpp:308-625): the whole forward pass on the device,
 * field build included.  raw_samples = sample_surface of the object. */
int lg_run_batch(lg_ctx* ctx, const lg_hand_desc* hand,
                 const lg_patches_desc* patches, const double* raw_samples,
                 int n_raw, const lg_run_params* params, lg_result** out);
/* Same, reusing a field built with lg_field_build (the cached-field mode). */
int lg_run_batch_field(lg_ctx* ctx, const lg_hand_desc* hand,
                       const lg_patches_desc* patches, lg_field* field,
                       const double* raw_samples, int n_raw,
                       const lg_run_params* params, lg_result** out);

/* ---- multi-GPU -------------------------------------------
 * Seed sharding: rank r of R calls lg_run_batch with shard_rank = r,
 * shard_count = R on its own context/GPU (candidates [rB/R, (r+1)B/R)); the
 * shards are independent and their union is the single-GPU result.  The only
 * collective is the final gather of the kept grasps to rank 0 over NCCL
 * (NVLink/NVSwitch inside a box).  It replaces the reference's parallel_for
 * over candidate chunks (parallel.hpp:24-56).  NCCL (libnccl.so.2) is bound at
 * run time by lg_comm_unique_id / lg_comm_init. */
#define LG_COMM_ID_BYTES 128
typedef struct lg_comm lg_comm;
/* Rank 0 creates the id; the caller distributes the bytes to every rank. */
int lg_comm_unique_id(unsigned char* id);
int lg_comm_init(lg_ctx* ctx, const unsigned char* id, int rank, int world, lg_comm** out);
void lg_comm_destroy(lg_comm* c);
/* Every rank passes its shard's kept grasps and profile.  Rank 0 receives all
 * grasps ordered by g (run_batch's kept order) in library-owned storage valid
 * until the next gather or lg_comm_destroy, and the merged profile (funnel
 * counts summed, stage seconds = max over ranks); other ranks get NULL / 0. */
int lg_comm_gather(lg_comm* c, const lg_grasp* grasps, long long n, const lg_profile* profile,
                   const lg_grasp** all, long long* n_all, lg_profile* merged);

#ifdef __cplusplus
}
#endif

#endif /* LG_H_ */
