"""Sharded decode-step hot path: one process per GPU.

Each rank computes its share of a VMM (giant steps g2 = rank mod world), of
QK^T (key ciphertexts j = rank mod world) or of Score*V (whole giant groups of
its baby-step / giant-step sum) through the C ABI's *_partial entry points; the
partial ciphertexts are all-gathered (NCCL over NVLink for device tensors; the
same code moves host tensors over gloo) and summed mod q on the GPU
(sf_sum_partials; NCCL has no mod-q reduction); the replicated tail (VMM
reduce ladder, Score*V lane fold) then runs on every rank. Modular addition is
exact and order-independent, so the result is bit-identical to one GPU.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional

import numpy as np

from . import Backend, Ciphertext, KVCache, VmmPlan, _check, _from_sf, _native, _to_sf
from ._native import SfLayout


# ------------------------------------------------------------------ ownership rules
GIANT_GROUPS = 8  # giants g2 = r mod 8 share one rotation sum


def own_giants(giants: int, rank: int, world: int) -> List[int]:
    """VMM giant steps a rank computes (csrc/protocols.cpp:vmm_partial): whole
    giant groups r = g2 mod GIANT_GROUPS with r mod world == rank (for world
    dividing 8 this is g2 mod world == rank)."""
    return [g for g in range(giants) if (g % GIANT_GROUPS) % world == rank]


PACK_GROUPS = 8  # key ciphertexts j = r mod 8 share one pack rotation sum


def own_keys(n_k: int, rank: int, world: int) -> List[int]:
    """K-cache ciphertexts a rank scores (csrc/protocols.cpp:qk_dot_partial):
    whole pack groups r = j mod PACK_GROUPS with r mod world == rank."""
    return [j for j in range(n_k) if (j % PACK_GROUPS) % world == rank]


SV_GROUPS = 8  # Score*V giants G = r mod 8 share one rotation sum


def sv_baby(n_variants: int) -> int:
    """Baby-step count B of the Score*V sum: the least power of two with B^2 >= #variants."""
    b = 1
    while b * b < n_variants:
        b <<= 1
    return b


def own_variants(n_variants: int, w_lo: int, w_hi: int, rank: int, world: int) -> List[int]:
    """Variants w of a cache group whose Score*V products a rank computes
    (csrc/protocols.cpp:softmax_times_v_partial): whole giant groups
    r = floor(w / B) mod SV_GROUPS with r mod world == rank."""
    B = sv_baby(n_variants)
    return [w for w in range(w_lo, w_hi) if ((w // B) % SV_GROUPS) % world == rank]


# --------------------------------------------------------------------- exchange
class _CudaArray:
    """__cuda_array_interface__ view of library-owned device words."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i8", "data": (ptr, False), "version": 3}


def ct_meta(ct: Ciphertext):
    lvl, sc, z, ly = ct._info()
    return (lvl, sc, z, ly)


def ct_device_words(ct: Ciphertext):
    """(c0_ptr, c1_ptr, words_per_poly) of a ciphertext's device buffer."""
    c0, c1, w = _native.u64p(), _native.u64p(), C.c_size_t()
    _check(_native.lib().sf_ct_device_view(ct.h, C.byref(c0), C.byref(c1), C.byref(w)))
    return C.cast(c0, C.c_void_p).value, C.cast(c1, C.c_void_p).value, w.value


def ct_from_device(be: Backend, c0_ptr: int, c1_ptr: int, meta) -> Ciphertext:
    lvl, sc, z, ly = meta
    s = _to_sf(ly)
    out = C.c_void_p()
    _check(_native.lib().sf_ct_from_device(be.ctx, c0_ptr, c1_ptr, lvl, sc, int(z), C.byref(s) if s else None,
                                            C.byref(out)))
    return Ciphertext(be, out.value)


def allgather_cts(be: Backend, cts: List[Ciphertext], group=None) -> List[List[Ciphertext]]:
    """All-gather a list of same-shape ciphertexts from every rank over NCCL.
    Returns [rank][i] handles (this rank's own entries are the inputs)."""
    import torch
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    metas = [ct_meta(c) for c in cts]
    all_meta: list = [None] * world
    dist.all_gather_object(all_meta, metas, group=group)
    be.synchronize()  # library stream -> torch stream ordering
    words = []
    for c in cts:
        c0, c1, w = ct_device_words(c)
        words.append(torch.as_tensor(_CudaArray(c0, w), device="cuda"))
        words.append(torch.as_tensor(_CudaArray(c1, w), device="cuda"))
    send = torch.cat(words)
    recv = torch.empty((world, send.numel()), dtype=send.dtype, device=send.device)
    dist.all_gather_into_tensor(recv, send, group=group)
    torch.cuda.synchronize()
    out = []
    for r in range(world):
        if r == rank:
            out.append(list(cts))
            continue
        row, off, got = recv[r], 0, []
        for m in all_meta[r]:
            w = (m[0] + 1) * be.n
            base = row.data_ptr()
            got.append(ct_from_device(be, base + off * 8, base + (off + w) * 8, m))
            off += 2 * w
        out.append(got)
    be.synchronize()  # copies out of `recv` complete before it is freed
    return out


# ---------------------------------------------------------------- sharded ops
def _ct(be: Backend, fn, *args) -> Ciphertext:
    out = C.c_void_p()
    _check(fn(be.ctx, *args, C.byref(out)))
    return Ciphertext(be, out.value)


def vmm_partial(be: Backend, x: Ciphertext, plan: VmmPlan, rank: int, world: int) -> Ciphertext:
    return _ct(be, _native.lib().sf_vmm_partial, x.h, plan.h, rank, world)


def vmm_finish(be: Backend, acc: Ciphertext, plan: VmmPlan, mask_output: bool = False) -> Ciphertext:
    return _ct(be, _native.lib().sf_vmm_finish, acc.h, plan.h, int(mask_output))


def sum_partials(be: Backend, parts: List[Ciphertext]) -> Ciphertext:
    arr = (C.c_void_p * len(parts))(*[p.h for p in parts])
    return _ct(be, _native.lib().sf_sum_partials, arr, len(parts))


def vmm_multi_partial(be: Backend, x: Ciphertext, plans, rank: int, world: int) -> List[Ciphertext]:
    k = len(plans)
    arr = (C.c_void_p * k)(*[p.h for p in plans])
    outs = (C.c_void_p * k)()
    _check(_native.lib().sf_vmm_multi_partial(be.ctx, x.h, arr, k, rank, world, outs))
    return [Ciphertext(be, outs[i]) for i in range(k)]


def vmm_multi_finish(be: Backend, accs: List[Ciphertext], plans, mask_output: bool = False) -> List[Ciphertext]:
    k = len(plans)
    a = (C.c_void_p * k)(*[x.h for x in accs])
    arr = (C.c_void_p * k)(*[p.h for p in plans])
    outs = (C.c_void_p * k)()
    _check(_native.lib().sf_vmm_multi_finish(be.ctx, a, arr, k, int(mask_output), outs))
    return [Ciphertext(be, outs[i]) for i in range(k)]


def qk_dot_partial(be: Backend, q: Ciphertext, cache: KVCache, rank: int, world: int) -> List[Ciphertext]:
    gt = cache.cfg.group_tokens
    cap = max(1, (max(cache.n_prime, 1) + gt - 1) // gt)
    maps = (C.c_void_p * cap)()
    n = C.c_int()
    _check(_native.lib().sf_qk_dot_partial(be.ctx, q.h, cache.h, rank, world, maps, C.byref(n)))
    return [Ciphertext(be, maps[i]) for i in range(n.value)]


def softmax_times_v_partial(be: Backend, probs, cache: KVCache, rank: int, world: int) -> List[Ciphertext]:
    """The rank's share of the baby-step / giant-step Score*V sum (one ciphertext)."""
    arr = (C.c_void_p * len(probs))(*[p.h for p in probs])
    return [_ct(be, _native.lib().sf_softmax_times_v_partial, arr, len(probs), cache.h, rank, world)]


def softmax_times_v_finish(be: Backend, parts: List[List[Ciphertext]], cache: KVCache) -> Ciphertext:
    """Sum the ranks' partials, fold the lanes, mask."""
    a = (C.c_void_p * len(parts))(*[p[0].h for p in parts])
    return _ct(be, _native.lib().sf_softmax_times_v_finish, a, len(parts), cache.h)


class Sharded:
    """The three sharded hot-path operators over a torch.distributed group."""

    def __init__(self, be: Backend, group=None):
        import torch.distributed as dist
        self.be, self.group = be, group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        be.set_value_shard(self.rank, self.world)

    def vmm(self, x: Ciphertext, plan: VmmPlan, mask_output: bool = False) -> Ciphertext:
        part = vmm_partial(self.be, x, plan, self.rank, self.world)
        parts = [p[0] for p in allgather_cts(self.be, [part], self.group)]
        return vmm_finish(self.be, sum_partials(self.be, parts), plan, mask_output)

    def vmm_multi(self, x: Ciphertext, plans, mask_output: bool = False) -> List[Ciphertext]:
        parts = vmm_multi_partial(self.be, x, plans, self.rank, self.world)
        got = allgather_cts(self.be, parts, self.group)
        accs = [sum_partials(self.be, [got[r][i] for r in range(self.world)]) for i in range(len(plans))]
        return vmm_multi_finish(self.be, accs, plans, mask_output)

    def qk_dot(self, q: Ciphertext, cache: KVCache) -> List[Ciphertext]:
        maps = qk_dot_partial(self.be, q, cache, self.rank, self.world)
        got = allgather_cts(self.be, maps, self.group)
        return [sum_partials(self.be, [got[r][m] for r in range(self.world)]) for m in range(len(maps))]

    def softmax_times_v(self, probs, cache: KVCache) -> Ciphertext:
        part = softmax_times_v_partial(self.be, probs, cache, self.rank, self.world)
        return softmax_times_v_finish(self.be, allgather_cts(self.be, part, self.group), cache)


class StreamSharded:
    """The sharded operators with the exchange on the library stream
    (csrc/comm.cpp): NCCL's all-gather is issued on the context stream, so a
    sharded step has no host synchronisation and can be captured whole into a
    CUDA graph (Backend.capture). The communicator is bootstrapped over the
    torch.distributed group (rank 0's NCCL unique id is broadcast); run each
    step once eagerly before capturing it (the exchange caches the call sites'
    ciphertext metadata on that first call)."""

    def __init__(self, be: Backend, group=None):
        import torch.distributed as dist
        self.be, self.group = be, group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        uid = C.create_string_buffer(128)
        if self.rank == 0:
            _check(_native.lib().sf_comm_unique_id(uid))
        box = [uid.raw]
        dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        _check(_native.lib().sf_comm_init(be.ctx, box[0], self.rank, self.world))

    def close(self) -> None:
        _check(_native.lib().sf_comm_destroy(self.be.ctx))

    def vmm(self, x: Ciphertext, plan: VmmPlan, mask_output: bool = False) -> Ciphertext:
        return _ct(self.be, _native.lib().sf_vmm_sharded, x.h, plan.h, int(mask_output))

    def vmm_multi(self, x: Ciphertext, plans, mask_output: bool = False) -> List[Ciphertext]:
        k = len(plans)
        arr = (C.c_void_p * k)(*[p.h for p in plans])
        outs = (C.c_void_p * k)()
        _check(_native.lib().sf_vmm_multi_sharded(self.be.ctx, x.h, arr, k, int(mask_output), outs))
        return [Ciphertext(self.be, outs[i]) for i in range(k)]

    def qk_dot(self, q: Ciphertext, cache: KVCache) -> List[Ciphertext]:
        gt = cache.cfg.group_tokens
        cap = max(1, (max(cache.n_prime, 1) + gt - 1) // gt)
        maps = (C.c_void_p * cap)()
        n = C.c_int()
        _check(_native.lib().sf_qk_dot_sharded(self.be.ctx, q.h, cache.h, maps, C.byref(n)))
        return [Ciphertext(self.be, maps[i]) for i in range(n.value)]

    def softmax_times_v(self, probs, cache: KVCache) -> Ciphertext:
        arr = (C.c_void_p * len(probs))(*[p.h for p in probs])
        return _ct(self.be, _native.lib().sf_softmax_times_v_sharded, arr, len(probs), cache.h)


class PeerSharded(StreamSharded):
    """The sharded operators with the exchange over peer memory
    (csrc/p2p.cu): every rank publishes its partial ciphertexts into a
    symmetric buffer exported with CUDA IPC, and one kernel per exchange reads
    all ranks' partials over NVLink and sums them mod q (the all-gather and the
    mod-add fused; no collective library). The IPC handles travel once over
    the torch.distributed group. `cap_words` sizes each of the two slots (the
    largest exchange of a decode step at ring 2^16 is two degree-2 Score*V
    parts at 3 limbs: ~1.6 M words)."""

    def __init__(self, be: Backend, group=None, cap_words: int = 1 << 21):
        import torch.distributed as dist
        self.be, self.group = be, group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        h = C.create_string_buffer(64)
        _check(_native.lib().sf_p2p_init(be.ctx, self.rank, self.world, cap_words, h))
        got: list = [None] * self.world
        dist.all_gather_object(got, h.raw, group=group)
        _check(_native.lib().sf_p2p_open(be.ctx, b"".join(got), self.world))

    def close(self) -> None:
        """Free the symmetric buffer once every rank is done reading it."""
        import torch.distributed as dist
        self.be.synchronize()
        dist.barrier(group=self.group)
        _check(_native.lib().sf_p2p_destroy(self.be.ctx))
