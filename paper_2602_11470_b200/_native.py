"""ctypes binding of libsf_b200.so (include/sf_b200.h).

There is no fallback: importing the package on a machine without the built
library raises, and any call on a machine without a CUDA device fails with the
library's SF_ERR_CUDA status.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsf_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "sf_b200.h")


class SfLayout(C.Structure):
    _fields_ = [("valid", C.c_int), ("kind", C.c_int), ("d", C.c_int), ("t", C.c_int), ("offset", C.c_int),
                ("heads", C.c_int), ("deferred_mask", C.c_int)]


class SfParams(C.Structure):
    _fields_ = [("slots", C.c_int), ("L", C.c_int), ("log_n", C.c_int), ("alpha", C.c_int), ("q0_bits", C.c_int),
                ("scale_bits", C.c_int), ("special_bits", C.c_int), ("device", C.c_int), ("seed", C.c_uint64)]


class SfOpCounts(C.Structure):
    _fields_ = [("rotations", C.c_longlong), ("hoisted_rotations", C.c_longlong), ("ct_pt_mults", C.c_longlong),
                ("ct_ct_mults", C.c_longlong), ("additions", C.c_longlong), ("bootstraps", C.c_longlong)]


vp = C.c_void_p
ip = C.POINTER(C.c_int)
dp = C.POINTER(C.c_double)
u64p = C.POINTER(C.c_uint64)
vpp = C.POINTER(C.c_void_p)
st = C.c_int

SIGNATURES = {
    "sf_last_error": (C.c_char_p, []),
    "sf_profile_butterflies": (st, [vp, dp]),
    "sf_host_profile": (st, [C.c_char_p, C.c_int, C.c_int]),
    "sf_rotate_many": (st, [vp, vpp, C.c_int, C.c_int, vpp]),
    "sf_vmm_interleaved_multi": (st, [vp, vp, vpp, C.c_int, C.c_int, vpp]),
    "sf_vmm_interleaved_many": (st, [vp, vpp, C.c_int, vp, C.c_int, vpp]),
    "sf_vmm_batch_plan_create": (st, [vp, dp, C.c_int, C.c_int, C.c_int, C.c_int, vpp]),
    "sf_vmm_plan_create_from_file": (st, [vp, C.c_char_p, C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, vpp]),
    "sf_vmm_plan_save": (st, [vp, vp, C.c_char_p]),
    "sf_vmm_plan_load": (st, [vp, C.c_char_p, vpp]),
    "sf_ct_wire_size": (st, [vp, vp, C.POINTER(C.c_size_t)]),
    "sf_ct_serialize": (st, [vp, vp, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "sf_ct_deserialize": (st, [vp, C.c_char_p, C.c_size_t, vpp]),
    "sf_vmm_batch": (st, [vp, vp, vp, vpp]),
    "sf_inner_rotate": (st, [vp, vp, C.c_int, C.c_int, C.c_int, vpp]),
    "sf_rope_apply_batch": (st, [vp, vp, C.c_int, C.c_int, C.c_longlong, C.c_double, vpp]),
    "sf_prefill_scores": (st, [vp, vpp, C.c_int, vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, vpp,
                               vpp, C.c_int, ip]),
    "sf_prefill_attend": (st, [vp, vpp, C.c_int, vp, vpp, C.c_int, ip]),
    "sf_bench_ntt": (st, [vp, C.c_int, C.c_int, C.c_int, dp]),
    "sf_graph_capture_begin": (st, [vp]),
    "sf_graph_capture_end": (st, [vp, vpp]),
    "sf_graph_launch": (st, [vp, vp]),
    "sf_graph_kernel_launches": (C.c_longlong, [vp]),
    "sf_graph_destroy": (None, [vp]),
    "sf_mem_stats": (st, [vp, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
    "sf_mem_reserve": (st, [vp, C.c_size_t]),
    "sf_set_value_shard": (st, [vp, C.c_int, C.c_int]),
    "sf_key_stats": (st, [vp, ip, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
    "sf_ct_refill": (st, [vp, vp, u64p]),
    "sf_ct_stage": (st, [vp, vp, u64p, C.c_int]),
    "sf_ct_stage_wait": (st, [vp, C.c_int]),
    "sf_ct_stage_out": (st, [vp, vp, u64p, C.c_int]),
    "sf_context_create": (st, [C.POINTER(SfParams), vpp]),
    "sf_context_destroy": (None, [vp]),
    "sf_context_info": (st, [vp, ip, ip, ip, ip, ip, u64p]),
    "sf_synchronize": (st, [vp]),
    "sf_gen_rotation_keys": (st, [vp, ip, C.c_int]),
    "sf_secret_key_export": (st, [vp, u64p]),
    "sf_switching_key_export": (st, [vp, C.c_uint64, u64p]),
    "sf_galois_elt": (C.c_uint64, [vp, C.c_int]),
    "sf_ct_retain": (vp, [vp]),
    "sf_ct_release": (None, [vp]),
    "sf_ct_info": (st, [vp, ip, dp, ip, C.POINTER(SfLayout)]),
    "sf_ct_with_layout": (st, [vp, vp, C.POINTER(SfLayout), vpp]),
    "sf_ct_export": (st, [vp, vp, u64p]),
    "sf_ct_import": (st, [vp, u64p, C.c_int, C.c_double, C.c_int, C.POINTER(SfLayout), vpp]),
    "sf_encrypt": (st, [vp, dp, C.c_int, C.POINTER(SfLayout), C.c_uint64, C.c_int, vpp]),
    "sf_zeros": (st, [vp, C.c_int, vpp]),
    "sf_decrypt": (st, [vp, vp, dp]),
    "sf_encode": (st, [vp, dp, C.c_double, C.c_int, u64p]),
    "sf_add": (st, [vp, vp, vp, vpp]),
    "sf_sub": (st, [vp, vp, vp, vpp]),
    "sf_add_plain": (st, [vp, vp, dp, vpp]),
    "sf_mul": (st, [vp, vp, vp, vpp]),
    "sf_mul_plain": (st, [vp, vp, dp, vpp]),
    "sf_mac_plain": (st, [vp, vpp, dp, C.c_int, vpp]),
    "sf_rotate": (st, [vp, vp, C.c_int, C.c_int, vpp]),
    "sf_rotate_hoisted": (st, [vp, vp, ip, C.c_int, vpp]),
    "sf_level_drop": (st, [vp, vp, C.c_int, vpp]),
    "sf_bootstrap": (st, [vp, vp, C.c_int, vpp]),
    "sf_ledger_totals": (st, [vp, C.POINTER(SfOpCounts)]),
    "sf_ledger_phase_totals": (st, [vp, C.c_char_p, C.POINTER(SfOpCounts)]),
    "sf_ledger_reset": (st, [vp]),
    "sf_phase_push": (st, [vp, C.c_char_p]),
    "sf_phase_pop": (st, [vp]),
    "sf_vmm_plan_create": (st, [vp, dp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vpp]),
    "sf_vmm_plan_destroy": (None, [vp]),
    "sf_vmm_predict": (st, [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_longlong),
                            C.POINTER(C.c_longlong), ip]),
    "sf_vmm_interleaved": (st, [vp, vp, vp, C.c_int, vpp]),
    "sf_kv_create": (st, [vp, C.c_int, C.c_int, C.c_int, C.c_int, vpp]),
    "sf_kv_retain": (vp, [vp]),
    "sf_kv_release": (None, [vp]),
    "sf_kv_info": (st, [vp, ip, ip, ip, ip]),
    "sf_kv_get": (st, [vp, C.c_int, C.c_int, C.c_int, vpp]),
    "sf_kv_from_cts": (st, [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vpp, C.c_int, vpp, C.c_int, vpp]),
    "sf_rope_apply": (st, [vp, vp, C.c_int, C.c_int, C.c_longlong, C.c_double, vpp]),
    "sf_rope_prepare": (st, [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_longlong, C.c_double]),
    "sf_fused_extract_mask": (st, [vp, vp, dp, vpp]),
    "sf_k_append": (st, [vp, vp, vp, vpp]),
    "sf_make_v_pieces": (st, [vp, vp, vp, C.c_int, vpp]),
    "sf_v_append": (st, [vp, vp, vpp, C.c_int, vpp]),
    "sf_qk_dot": (st, [vp, vp, vp, vpp, ip]),
    "sf_softmax_times_v": (st, [vp, vpp, C.c_int, vp, vpp]),
    "sf_vmm_partial": (st, [vp, vp, vp, C.c_int, C.c_int, vpp]),
    "sf_vmm_finish": (st, [vp, vp, vp, C.c_int, vpp]),
    "sf_qk_dot_partial": (st, [vp, vp, vp, C.c_int, C.c_int, vpp, ip]),
    "sf_softmax_times_v_partial": (st, [vp, vpp, C.c_int, vp, C.c_int, C.c_int, vpp]),
    "sf_softmax_times_v_finish": (st, [vp, vpp, C.c_int, vp, vpp]),
    "sf_sum_partials": (st, [vp, vpp, C.c_int, vpp]),
    "sf_vmm_multi_partial": (st, [vp, vp, vpp, C.c_int, C.c_int, C.c_int, vpp]),
    "sf_vmm_multi_finish": (st, [vp, vpp, vpp, C.c_int, C.c_int, vpp]),
    "sf_vmm_multi_sharded": (st, [vp, vp, vpp, C.c_int, C.c_int, vpp]),
    "sf_p2p_init": (st, [vp, C.c_int, C.c_int, C.c_size_t, C.c_char_p]),
    "sf_p2p_open": (st, [vp, C.c_char_p, C.c_int]),
    "sf_p2p_destroy": (st, [vp]),
    "sf_comm_unique_id": (st, [C.c_char_p]),
    "sf_comm_init": (st, [vp, C.c_char_p, C.c_int, C.c_int]),
    "sf_comm_destroy": (st, [vp]),
    "sf_vmm_sharded": (st, [vp, vp, vp, C.c_int, vpp]),
    "sf_qk_dot_sharded": (st, [vp, vp, vp, vpp, ip]),
    "sf_softmax_times_v_sharded": (st, [vp, vpp, C.c_int, vp, vpp]),
    "sf_ct_device_view": (st, [vp, C.POINTER(u64p), C.POINTER(u64p), C.POINTER(C.c_size_t)]),
    "sf_ct_from_device": (st, [vp, C.c_void_p, C.c_void_p, C.c_int, C.c_double, C.c_int, C.POINTER(SfLayout), vpp]),
    "sf_event_record": (st, [vp, C.c_int]),
    "sf_event_elapsed_ms": (st, [vp, C.c_int, C.c_int, C.POINTER(C.c_float)]),
    "sf_kernel_launches": (C.c_longlong, [vp]),
    "sf_profile_begin": (st, [vp, C.c_int]),
    "sf_profile_end": (st, [vp, dp, dp, C.POINTER(C.c_longlong)]),
}

_lib = None


def build(verbose: bool = False) -> str:
    """Compile libsf_b200.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
    r = subprocess.run(["make", "-j8"], cwd=HERE, capture_output=not verbose, text=True)
    if r.returncode != 0:
        raise RuntimeError("libsf_b200 build failed:\n" + (r.stdout or "") + (r.stderr or ""))
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run paper_2602_11470_b200._native.build() "
                              "(no CPU fallback exists for the product path)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _lib = L
    return _lib


def declared_symbols():
    """Function names declared in include/sf_b200.h."""
    import re
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(sf_[a-z0-9_]+)\(", txt)))
