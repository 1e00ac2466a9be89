/*
 * lg_caller.h — the stand-in CALLER of the drop-in boundary (not the product).
 *
 * The reference keeps these steps on the host (SURVEY.md 8(b) "What stays"):
 * parse_config (config.cpp:339-417), load_mesh and the primitive meshes
 * (mesh.cpp:161-273), sample_surface (mesh.cpp:297-339), the hand's surface
 * samples + decompose_patches (pipeline.cpp:277-285, contact_field.cpp:26-99)
 * and write_dataset / write_profile (dataset.cpp:23-131).  A production
 * integration calls the reference's own functions for them;
 * this library restates them so the bench and the tests can drive
 * libgraspgen_b200.so without the reference tree.  Everything it returns is a
 * flat view in the include/lg.h layout.
 */
#ifndef LG_CALLER_H_
#define LG_CALLER_H_

#include "lg.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lgc_mesh lgc_mesh;
typedef struct lgc_patches lgc_patches;

typedef struct lgc_load_report {
  long long triangles_read, triangles_kept, degenerate_dropped;
} lgc_load_report;

int lgc_last_error(char* buf, size_t cap);

/* RunConfig defaults (config.hpp:15-77) and parse_config with CLI overrides. */
void lgc_run_params_default(lg_run_params* p);
int lgc_config_parse(const char* path, const char* hand, const char* object, const char* out,
                     const long long* seed, const int* batch, const int* workers,
                     lg_run_params* p);
/* index_cache_key (config.cpp:403-417): FNV-1a of the hand file and the
 * index-shaping parameters (the GGCF cache key). */
int lgc_index_cache_key(const lg_run_params* p, uint64_t* key);

/* TriMesh: load_mesh (mesh.cpp:161-167), make_box / make_icosphere /
 * make_cylinder (mesh.cpp:181-273), OBJ export. */
int lgc_mesh_load(const char* path, lgc_load_report* report, lgc_mesh** out);
int lgc_mesh_box(double sx, double sy, double sz, lgc_mesh** out);
int lgc_mesh_icosphere(double radius, int subdivisions, lgc_mesh** out);
int lgc_mesh_cylinder(double radius, double length, int segments, lgc_mesh** out);
int lgc_mesh_from_arrays(const double* verts, int n_verts, const int* tris, int n_tris,
                         lgc_mesh** out);
int lgc_mesh_scale(lgc_mesh* m, double scale);
int lgc_mesh_info(const lgc_mesh* m, int* n_verts, int* n_tris, double* area);
int lgc_mesh_arrays(const lgc_mesh* m, const double** verts, const int** tris);
int lgc_mesh_save_obj(const lgc_mesh* m, const char* path);
void lgc_mesh_destroy(lgc_mesh* m);

/* sample_surface (mesh.cpp:297-339) -> [n][6]; pass out=NULL for the count. */
int lgc_sample_surface(const lgc_mesh* m, double samples_per_cm2, uint64_t seed, double* out,
                       size_t cap, size_t* n);

/* build_field's host hand steps (pipeline.cpp:277-285) on the host. */
int lgc_hand_patches(const lg_hand_desc* hand, const lg_visual_desc* visual,
                     double samples_per_cm2, double patch_radius, uint64_t seed, int field_cap,
                     lgc_patches** out);
int lgc_patches_export(const lgc_patches* p, lg_patches_desc* out);
void lgc_patches_destroy(lgc_patches* p);

/* write_dataset JSONL (dataset.cpp:23-56) and the profile JSON (113-131). */
int lgc_write_dataset(const char* path, const lg_grasp* grasps, long long n);
int lgc_write_profile(const char* path, const lg_profile* p);

#ifdef __cplusplus
}
#endif

#endif /* LG_CALLER_H_ */
