"""ctypes mirror of include/lg.h (structs + prototypes).

Shared by the product wrapper (paper_2511_07418_b200/api.py) and, for the
struct layouts only, by the oracle binding under oracle/.
"""
import ctypes as C

LG_MAX_K = 5
LG_MAX_CONTACTS = 6
LG_MAX_DOF = 32
LG_MAX_GROUPS = 32
LG_COMM_ID_BYTES = 128

LG_OK = 0
LG_ERR_INVALID_ARGUMENT = -1
LG_ERR_RUNTIME = -2
LG_ERR_OUT_OF_RANGE = -3
LG_ERR_CUDA = -4
LG_ERR_NOMEM = -5

dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int)
llp = C.POINTER(C.c_longlong)


class HandDesc(C.Structure):
    _fields_ = [
        ("n_links", C.c_int), ("dof", C.c_int), ("root", C.c_int),
        ("parent", ip), ("joint_type", ip), ("joint_index", ip), ("topo_order", ip),
        ("origin_R", dp), ("origin_t", dp), ("axis", dp), ("limit_lo", dp), ("limit_hi", dp),
        ("n_parts", C.c_int), ("part_link", ip), ("part_vert_off", ip), ("part_verts", dp),
        ("part_tri_off", ip), ("part_tris", ip), ("part_plane_off", ip), ("part_planes", dp),
        ("part_bounds", dp),
    ]


class PatchesDesc(C.Structure):
    _fields_ = [
        ("n_patches", C.c_int), ("link", ip), ("point_off", ip), ("points", dp),
        ("normals", dp), ("fp_off", ip), ("field_points", ip),
    ]


class FieldCsr(C.Structure):
    _fields_ = [
        ("box_width", C.c_double), ("codebook_size", C.c_int), ("codebook", dp),
        ("n_patches", C.c_int), ("patch_link", ip), ("patch_box_off", ip),
        ("n_boxes", C.c_longlong), ("box_cell", llp), ("box_code_off", llp),
        ("n_codes", C.c_longlong), ("codes", C.POINTER(C.c_uint16)), ("rep_link", ip),
        ("rep_point", dp), ("rep_normal", dp), ("n_vectors", C.c_longlong),
    ]


class RunParams(C.Structure):
    _fields_ = [
        ("hand", C.c_char * 512), ("object", C.c_char * 512), ("out", C.c_char * 512),
        ("seed", C.c_uint64),
        ("batch", C.c_int), ("workers", C.c_int), ("passes", C.c_int), ("cache", C.c_int),
        ("export_obj", C.c_int), ("k_contacts", C.c_int),
        ("samples_per_cm2", C.c_double), ("object_scale", C.c_double),
        ("probe_half_width", C.c_double), ("probe_depth_threshold", C.c_double),
        ("hand_scale", C.c_double),
        ("field_configs", C.c_int),
        ("box_width", C.c_double), ("patch_radius", C.c_double),
        ("field_points_per_patch", C.c_int), ("codebook_size", C.c_int),
        ("theta_hit", C.c_double),
        ("placement_mode", C.c_int),
        ("static_contact_prob", C.c_double),
        ("canonical_center", C.c_double * 3), ("canonical_half_extents", C.c_double * 3),
        ("penetration_margin", C.c_double),
        ("lambda_torque", C.c_double), ("mu", C.c_double), ("eps_stable", C.c_double),
        ("pgd_iterations", C.c_int), ("pgd_warm_iterations", C.c_int),
        ("pgd_step", C.c_double),
        ("n_outer", C.c_int), ("n_inner", C.c_int), ("restarts", C.c_int),
        ("sigma", C.c_double), ("beta", C.c_double),
        ("ik_iterations", C.c_int),
        ("step_clamp", C.c_double), ("residual_tol", C.c_double), ("damping_scale", C.c_double),
        ("finetune_rounds", C.c_int), ("finetune_iterations", C.c_int),
        ("lookup_attempts", C.c_int), ("unused_attempts", C.c_int),
        ("contact_tol", C.c_double),
        ("shard_rank", C.c_int), ("shard_count", C.c_int), ("want_trace", C.c_int),
    ]


class Grasp(C.Structure):
    _fields_ = [
        ("g", C.c_longlong), ("pose_R", C.c_double * 9), ("pose_t", C.c_double * 3),
        ("dof", C.c_int), ("q", C.c_double * LG_MAX_DOF), ("n_contacts", C.c_int),
        ("contact_p", (C.c_double * 3) * LG_MAX_CONTACTS),
        ("contact_n", (C.c_double * 3) * LG_MAX_CONTACTS),
        ("contact_link", C.c_int * LG_MAX_CONTACTS), ("objective", C.c_double),
        ("penetration_free", C.c_int), ("stable", C.c_int), ("ik_converged", C.c_int),
    ]


class Profile(C.Structure):
    _fields_ = [(n, C.c_double) for n in (
        "placement_domains", "contact_optimization", "kinematics_optimization",
        "postprocessing", "total", "field_build")] + [(n, C.c_longlong) for n in (
        "candidates", "placements_accepted", "contact_sets_balanced", "ik_finite",
        "penetration_free", "ik_converged", "stable", "valid")] + [
        ("grasps_per_second", C.c_double)] + [(n, C.c_longlong) for n in (
        "patches", "boxes", "field_vectors", "object_samples", "field_samples", "gpu_launches")] + [
        ("device_seconds", C.c_double), ("h2d_bytes", C.c_longlong),
        ("d2h_bytes", C.c_longlong)] + [(n, C.c_longlong) for n in (
        "ik_iterations", "fk_evals", "wrench_evals", "wrench_grads", "proj_evals",
        "realize_calls", "collision_calls")] + [
        ("realize_seconds", C.c_double), ("contact_opt_seconds", C.c_double),
        ("index_from_cache", C.c_longlong), ("index_codes", C.c_longlong)]


class GraspCheck(C.Structure):
    """lg_grasp_check: validate_dataset's measured quantities per grasp."""
    _fields_ = [
        ("status", C.c_int), ("rigid_error", C.c_double), ("n_limit", C.c_int),
        ("limit_link", C.c_int * LG_MAX_DOF), ("limit_value", C.c_double * LG_MAX_DOF),
        ("n_contacts", C.c_int), ("contact_state", C.c_int * LG_MAX_CONTACTS),
        ("hand_dist", C.c_double * LG_MAX_CONTACTS), ("object_dist", C.c_double * LG_MAX_CONTACTS),
        ("worst_depth", C.c_double), ("wrench_error", C.c_int), ("wrench_objective", C.c_double),
    ]


class Trace(C.Structure):
    _fields_ = [
        ("g", C.c_longlong), ("pass_", C.c_int), ("c", C.c_int),
        ("accepted", C.c_int), ("penetration", C.c_double),
        ("pose_R", C.c_double * 9), ("pose_t", C.c_double * 3),
        ("n_static", C.c_int), ("static_link", C.c_int),
        ("static_p", C.c_double * 3), ("static_n", C.c_double * 3),
        ("n_groups", C.c_int), ("domain_size", C.c_int * LG_MAX_GROUPS),
        ("picked", C.c_int), ("chosen", C.c_int * LG_MAX_K),
        ("opt_element", C.c_int * LG_MAX_K), ("opt_sample", C.c_int * LG_MAX_K),
        ("opt_objective", C.c_double), ("opt_anchor", C.c_int), ("opt_evaluations", C.c_int),
        ("opt_alpha", C.c_double * LG_MAX_CONTACTS), ("opt_bx", C.c_double * LG_MAX_CONTACTS),
        ("opt_by", C.c_double * LG_MAX_CONTACTS),
        ("balanced", C.c_int),
        ("realized", C.c_int), ("attempts_run", C.c_int), ("best_attempt", C.c_int),
        ("best_clear", C.c_int), ("max_residual", C.c_double),
        ("real_q", C.c_double * LG_MAX_DOF), ("used_joints", C.c_ulonglong),
        ("target_link", C.c_int * LG_MAX_K),
        ("target_point", (C.c_double * 3) * LG_MAX_K),
        ("target_normal", (C.c_double * 3) * LG_MAX_K),
        ("unused_attempt", C.c_int), ("penetration_free", C.c_int), ("ik_converged", C.c_int),
        ("stable", C.c_int), ("valid", C.c_int), ("dropped", C.c_int),
        ("final_q", C.c_double * LG_MAX_DOF), ("objective", C.c_double),
    ]


class LoadReport(C.Structure):
    _fields_ = [("triangles_read", C.c_longlong), ("triangles_kept", C.c_longlong),
                ("degenerate_dropped", C.c_longlong)]


# numpy structured dtypes with identical layouts (for zero-copy views)
def _np_dtype(struct):
    import numpy as np
    names, formats, offsets = [], [], []
    for name, ctype in struct._fields_:
        names.append(name)
        formats.append(np.dtype(ctype))
        offsets.append(getattr(struct, name).offset)
    return np.dtype({"names": names, "formats": formats, "offsets": offsets,
                     "itemsize": C.sizeof(struct)})


def grasp_dtype():
    return _np_dtype(Grasp)


def check_dtype():
    return _np_dtype(GraspCheck)


def trace_dtype():
    return _np_dtype(Trace)
