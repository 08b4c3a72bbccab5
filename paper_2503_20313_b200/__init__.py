"""B200-native TileLink tensor-parallel MLP hot path (arXiv 2503.20313).

Thin Python binding over the C ABI in include/tl_api.h.  PyTorch is used only for device
memory, streams and process groups; every step of AG-GEMM / GEMM-RS / MLP runs in the
library's sm_100a kernels.  There is no CPU fallback: without the built library or an sm_100
device every compute call raises.
"""
from __future__ import annotations

import ctypes as C

from ._lib import TLError, check, lib, ptr_array

ACT_NONE, ACT_SILU_MUL, ACT_GELU_TANH_MUL = 0, 1, 2
ACTS = {"none": ACT_NONE, "silu_mul": ACT_SILU_MUL, "gelu_tanh_mul": ACT_GELU_TANH_MUL}

__all__ = ["Comm", "TLError", "lib", "ACT_NONE", "ACT_SILU_MUL", "ACT_GELU_TANH_MUL", "static_map_device",
           "moe_capacity", "moe_ag_gemm", "moe_ag_gemm_lb", "moe_gemm_rs", "moe_gemm_rs_lb", "sp_attention",
           "sp_attention_lb"]


def _ptr(t):
    return None if t is None else t.data_ptr()


def _stream(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _bf16(t, name):
    import torch
    if t.dtype != torch.bfloat16 or not t.is_cuda or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous bf16 CUDA tensor")
    return t


def _dev(t, name, dtype, shape, device=None):
    """Argument check before a pointer crosses the C ABI (which cannot see dtypes or memory kinds):
    a contiguous CUDA tensor of `dtype` on `device` whose shape is `shape` (None entries: any)."""
    import torch
    if t is None:
        return None
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if t.dtype != dtype or not t.is_cuda or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous {dtype} CUDA tensor (got {t.dtype}, "
                         f"{'cuda' if t.is_cuda else t.device.type}, contiguous={t.is_contiguous()})")
    if device is not None and t.device.index != device:
        raise ValueError(f"{name} is on cuda:{t.device.index}, the comm on cuda:{device}")
    if len(t.shape) != len(shape) or any(e is not None and e != g for e, g in zip(shape, t.shape)):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple('*' if e is None else e for e in shape)}")
    return t


def _check_ag(world, dev, A_shard, B, C_out, A_gathered, act):
    import torch
    bf = torch.bfloat16
    _dev(A_shard, "A_shard", bf, (None, None), dev)
    Mr, K = A_shard.shape
    _dev(C_out, "C", bf, (Mr * world, None), dev)
    N = C_out.shape[1]
    _dev(B, "B", bf, (N * (1 if act == ACT_NONE else 2), K), dev)
    _dev(A_gathered, "A_gathered", bf, (Mr * world, K), dev)


def _check_rs(world, dev, A, B, C_shard):
    import torch
    bf = torch.bfloat16
    _dev(A, "A", bf, (None, None), dev)
    M, K = A.shape
    _dev(B, "B", bf, (None, K), dev)
    if M % world:
        raise ValueError(f"A has {M} rows, not divisible by world={world}")
    _dev(C_shard, "C_shard", bf, (M // world, B.shape[0]), dev)


def _check_mlp(world, dev, X_shard, W1, W2, out, Z, act):
    import torch
    bf = torch.bfloat16
    _dev(X_shard, "X_shard", bf, (None, None), dev)
    Mr, H = X_shard.shape
    _dev(W2, "W2", bf, (H, None), dev)
    Il = W2.shape[1]
    _dev(W1, "W1", bf, (Il * (1 if act == ACT_NONE else 2), H), dev)
    _dev(out, "out_shard", bf, (Mr, H), dev)
    _dev(Z, "Z", bf, (Mr * world, Il), dev)


def _same_len(world, **lists):
    for n, L in lists.items():
        if L is not None and len(L) != world:
            raise ValueError(f"{n}: {len(L)} tensors for a {world}-rank loopback comm")


class Comm:
    """A TileLink communicator: symmetric workspace + epochs (tl_comm_t)."""

    def __init__(self, handle, rank, world, local_ranks, device):
        self._h = C.c_void_p(handle)
        self.rank, self.world, self.local_ranks, self.device = rank, world, local_ranks, device

    # ------------------------------------------------------------------ construction
    @classmethod
    def loopback(cls, world: int, device: int = 0, max_M: int = 8192, max_H: int = 4096, max_topk: int = 1):
        """All `world` ranks emulated on one device, driven by single launches."""
        L = lib()
        h = C.c_void_p()
        check(L.tl_comm_create_loopback_ex(world, device, max_M, max_H, max_topk, C.byref(h)),
              "tl_comm_create_loopback_ex")
        return cls(h.value, -1, world, world, device)

    @classmethod
    def single(cls, device: int = 0, max_M: int = 8192, max_H: int = 4096, max_topk: int = 1):
        """World of one rank (AG/RS degenerate to identities)."""
        L = lib()
        h = C.c_void_p()
        buf = C.create_string_buffer(L.tl_handle_size())
        check(L.tl_comm_create_ex(0, 1, device, max_M, max_H, max_topk, buf, C.byref(h)), "tl_comm_create_ex")
        return cls(h.value, 0, 1, 1, device)

    @classmethod
    def from_process_group(cls, group=None, device: int | None = None, max_M: int = 8192, max_H: int = 4096,
                           max_topk: int = 1):
        """One process per GPU: create, all-gather the IPC handles over `group`, connect."""
        import torch
        import torch.distributed as dist
        from .bootstrap import exchange_handles
        L = lib()
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        if device is None:
            device = torch.cuda.current_device()
        h = C.c_void_p()
        buf = C.create_string_buffer(L.tl_handle_size())
        check(L.tl_comm_create_ex(rank, world, device, max_M, max_H, max_topk, buf, C.byref(h)), "tl_comm_create_ex")
        comm = cls(h.value, rank, world, 1, device)
        if world > 1:
            allh = exchange_handles(bytes(buf.raw), group)
            check(L.tl_comm_connect(comm._h, C.create_string_buffer(allh, len(allh))), "tl_comm_connect")
            dist.barrier(group)
        return comm

    def close(self):
        if self._h is not None and self._h.value:
            lib().tl_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ options / diag
    def set_option(self, key: str, value: int):
        check(lib().tl_set_option(self._h, key.encode(), int(value)), "tl_set_option")

    def get_option(self, key: str) -> int:
        v = C.c_int64()
        check(lib().tl_get_option(self._h, key.encode(), C.byref(v)), "tl_get_option")
        return v.value

    def check(self):
        """(status, diag[8]) after synchronising the device (tl_comm_check)."""
        d = (C.c_int64 * 8)()
        st = lib().tl_comm_check(self._h, d)
        return st, list(d)

    # ------------------------------------------------------------------ ops (one rank per process)
    def ag_gemm(self, A_shard, B, C_out, A_gathered=None, act: int = ACT_NONE, stream=None):
        _check_ag(self.world, self.device, A_shard, B, C_out, A_gathered, act)
        M = A_shard.shape[0] * self.world
        K = A_shard.shape[1]
        N = C_out.shape[1]
        check(lib().tl_ag_gemm_act(self._h, _ptr(A_shard), _ptr(B), _ptr(C_out), _ptr(A_gathered), M, N, K, act,
                                   _stream(stream)), "tl_ag_gemm_act")
        return C_out

    def gemm_rs(self, A, B, C_shard, stream=None):
        _check_rs(self.world, self.device, A, B, C_shard)
        M, K = A.shape
        N = B.shape[0]
        check(lib().tl_gemm_rs(self._h, _ptr(A), _ptr(B), _ptr(C_shard), M, N, K, _stream(stream)), "tl_gemm_rs")
        return C_shard

    def mlp_forward(self, X_shard, W1, W2, out_shard, act: int = ACT_SILU_MUL, Z=None, stream=None):
        _check_mlp(self.world, self.device, X_shard, W1, W2, out_shard, Z, act)
        M = X_shard.shape[0] * self.world
        H = X_shard.shape[1]
        I_l = W2.shape[1]
        check(lib().tl_mlp_forward(self._h, _ptr(X_shard), _ptr(W1), _ptr(W2), _ptr(out_shard), _ptr(Z), M, H, I_l,
                                   act, _stream(stream)), "tl_mlp_forward")
        return out_shard

    # ------------------------------------------------------------------ ops (loopback: lists per rank)
    def ag_gemm_lb(self, A_shards, Bs, Cs, A_gathered=None, act: int = ACT_NONE, stream=None):
        W = self.world
        _same_len(W, A_shards=A_shards, Bs=Bs, Cs=Cs, A_gathered=A_gathered)
        for i in range(W):
            _check_ag(W, self.device, A_shards[i], Bs[i], Cs[i], A_gathered[i] if A_gathered else None, act)
        M = A_shards[0].shape[0] * W
        K = A_shards[0].shape[1]
        N = Cs[0].shape[1]
        a, _ka = ptr_array([_ptr(t) for t in A_shards])
        b, _kb = ptr_array([_ptr(t) for t in Bs])
        c, _kc = ptr_array([_ptr(t) for t in Cs])
        g, _kg = ptr_array([_ptr(t) for t in A_gathered]) if A_gathered is not None else (None, None)
        check(lib().tl_ag_gemm_loopback(self._h, a, b, c, g, M, N, K, act, _stream(stream)), "tl_ag_gemm_loopback")
        return Cs

    def gemm_rs_lb(self, As, Bs, Cs, stream=None):
        _same_len(self.world, As=As, Bs=Bs, Cs=Cs)
        for i in range(self.world):
            _check_rs(self.world, self.device, As[i], Bs[i], Cs[i])
        M, K = As[0].shape
        N = Bs[0].shape[0]
        a, _ka = ptr_array([_ptr(t) for t in As])
        b, _kb = ptr_array([_ptr(t) for t in Bs])
        c, _kc = ptr_array([_ptr(t) for t in Cs])
        check(lib().tl_gemm_rs_loopback(self._h, a, b, c, M, N, K, _stream(stream)), "tl_gemm_rs_loopback")
        return Cs

    def mlp_forward_lb(self, X_shards, W1s, W2s, outs, act: int = ACT_SILU_MUL, Zs=None, stream=None):
        W = self.world
        _same_len(W, X_shards=X_shards, W1s=W1s, W2s=W2s, outs=outs, Zs=Zs)
        for i in range(W):
            _check_mlp(W, self.device, X_shards[i], W1s[i], W2s[i], outs[i], Zs[i] if Zs else None, act)
        M = X_shards[0].shape[0] * W
        H = X_shards[0].shape[1]
        I_l = W2s[0].shape[1]
        x, _kx = ptr_array([_ptr(t) for t in X_shards])
        w1, _k1 = ptr_array([_ptr(t) for t in W1s])
        w2, _k2 = ptr_array([_ptr(t) for t in W2s])
        o, _ko = ptr_array([_ptr(t) for t in outs])
        z, _kz = ptr_array([_ptr(t) for t in Zs]) if Zs is not None else (None, None)
        check(lib().tl_mlp_forward_loopback(self._h, x, w1, w2, o, z, M, H, I_l, act, _stream(stream)),
              "tl_mlp_forward_loopback")
        return outs


def _check_moe_ag(comm, X_shard, topk_ids, W1, Y, row_ids, offsets, act):
    import torch
    bf, dev = torch.bfloat16, comm.device
    _dev(X_shard, "X_shard", bf, (None, None), dev)
    Mr, H = X_shard.shape
    _dev(topk_ids, "topk_ids", torch.int32, (Mr * comm.world, None), dev)
    _dev(W1, "W1", bf, (None, None, H), dev)
    E, topk = W1.shape[0], topk_ids.shape[1]
    R = moe_capacity(comm, Mr * comm.world, topk, E)
    _dev(Y, "Y", bf, (R, W1.shape[1] // (1 if act == ACT_NONE else 2)), dev)
    _dev(row_ids, "row_ids", torch.int32, (R,), dev)
    _dev(offsets, "offsets", torch.int32, (E + 1,), dev)


def _check_moe_rs(comm, Zg, row_ids, offsets, topk_weights, W2, out_shard):
    import torch
    bf, dev = torch.bfloat16, comm.device
    _dev(topk_weights, "topk_weights", torch.float32, (None, None), dev)
    M, topk = topk_weights.shape
    _dev(W2, "W2", bf, (None, None, None), dev)
    E, H, Il = W2.shape
    R = moe_capacity(comm, M, topk, E)
    _dev(Zg, "Zg", bf, (R, Il), dev)
    _dev(row_ids, "row_ids", torch.int32, (R,), dev)
    _dev(offsets, "offsets", torch.int32, (E + 1,), dev)
    if M % comm.world:
        raise ValueError(f"{M} tokens not divisible by world={comm.world}")
    _dev(out_shard, "out_shard", bf, (M // comm.world, H), dev)


def moe_capacity(comm, M: int, topk: int, E: int) -> int:
    return lib().tl_moe_capacity(comm._h, M, topk, E)


def moe_ag_gemm(comm, X_shard, topk_ids, W1, Y, row_ids, offsets, act: int = ACT_SILU_MUL, stream=None):
    """MoE AG + Gather + GroupGEMM on a one-rank-per-process comm (see tl_api.h)."""
    _check_moe_ag(comm, X_shard, topk_ids, W1, Y, row_ids, offsets, act)
    M = X_shard.shape[0] * comm.world
    H = X_shard.shape[1]
    E, topk = W1.shape[0], topk_ids.shape[1]
    N_out = Y.shape[1]
    check(lib().tl_moe_ag_gemm(comm._h, _ptr(X_shard), _ptr(topk_ids), _ptr(W1), _ptr(Y), _ptr(row_ids),
                               _ptr(offsets), M, H, N_out, E, topk, act, _stream(stream)), "tl_moe_ag_gemm")
    return Y


def moe_ag_gemm_lb(comm, X_shards, topk_ids, W1s, Ys, row_ids, offsets, act: int = ACT_SILU_MUL, stream=None):
    """Loopback variant: per-rank lists (topk_ids / row_ids / offsets are per-rank device copies)."""
    W = comm.world
    _same_len(W, X_shards=X_shards, topk_ids=topk_ids, W1s=W1s, Ys=Ys, row_ids=row_ids, offsets=offsets)
    for i in range(W):
        _check_moe_ag(comm, X_shards[i], topk_ids[i], W1s[i], Ys[i], row_ids[i], offsets[i], act)
    M = X_shards[0].shape[0] * W
    H = X_shards[0].shape[1]
    E, topk = W1s[0].shape[0], topk_ids[0].shape[1]
    N_out = Ys[0].shape[1]
    arrs = [ptr_array([_ptr(t) for t in L]) for L in (X_shards, topk_ids, W1s, Ys, row_ids, offsets)]
    check(lib().tl_moe_ag_gemm_loopback(comm._h, *[a[0] for a in arrs], M, H, N_out, E, topk, act,
                                        _stream(stream)), "tl_moe_ag_gemm_loopback")
    return Ys


def moe_gemm_rs(comm, Zg, row_ids, offsets, topk_weights, W2, out_shard, stream=None):
    """MoE GroupGEMM + Scatter + TopK reduce + RS on a one-rank-per-process comm (see tl_api.h)."""
    _check_moe_rs(comm, Zg, row_ids, offsets, topk_weights, W2, out_shard)
    M, topk = topk_weights.shape
    E, H, I_l = W2.shape
    check(lib().tl_moe_gemm_rs(comm._h, _ptr(Zg), _ptr(row_ids), _ptr(offsets), _ptr(topk_weights), _ptr(W2),
                               _ptr(out_shard), M, H, I_l, E, topk, _stream(stream)), "tl_moe_gemm_rs")
    return out_shard


def moe_gemm_rs_lb(comm, Zgs, row_ids, offsets, topk_weights, W2s, outs, stream=None):
    _same_len(comm.world, Zgs=Zgs, row_ids=row_ids, offsets=offsets, topk_weights=topk_weights, W2s=W2s, outs=outs)
    for i in range(comm.world):
        _check_moe_rs(comm, Zgs[i], row_ids[i], offsets[i], topk_weights[i], W2s[i], outs[i])
    M, topk = topk_weights[0].shape
    E, H, I_l = W2s[0].shape
    arrs = [ptr_array([_ptr(t) for t in L]) for L in (Zgs, row_ids, offsets, topk_weights, W2s, outs)]
    check(lib().tl_moe_gemm_rs_loopback(comm._h, *[a[0] for a in arrs], M, H, I_l, E, topk, _stream(stream)),
          "tl_moe_gemm_rs_loopback")
    return outs


def sp_attention(comm, Q_shard, K_shard, V_shard, O_shard, scale: float | None = None, stream=None):
    """Sequence-parallel attention: AllGather(K, V) fused with flash attention (tl_sp_attention).
    Q/K/V/O shards: contiguous bf16 CUDA tensors [S/world, heads, 128]."""
    import torch
    _dev(Q_shard, "Q", torch.bfloat16, (None, None, None), comm.device)
    S_r, heads, D = Q_shard.shape
    for n, t in (("K", K_shard), ("V", V_shard), ("O", O_shard)):
        _dev(t, n, torch.bfloat16, (S_r, heads, D), comm.device)
    scale = D ** -0.5 if scale is None else scale
    check(lib().tl_sp_attention(comm._h, _ptr(Q_shard), _ptr(K_shard), _ptr(V_shard), _ptr(O_shard), S_r * comm.world,
                                heads, D, scale, _stream(stream)), "tl_sp_attention")
    return O_shard


def sp_attention_lb(comm, Qs, Ks, Vs, Os, scale: float | None = None, stream=None):
    """Loopback variant: per-rank lists of shards."""
    import torch
    _same_len(comm.world, Qs=Qs, Ks=Ks, Vs=Vs, Os=Os)
    S_r, heads, D = Qs[0].shape
    for n, L in (("Q", Qs), ("K", Ks), ("V", Vs), ("O", Os)):
        for t in L:
            _dev(t, n, torch.bfloat16, (S_r, heads, D), comm.device)
    scale = D ** -0.5 if scale is None else scale
    arrs = [ptr_array([_ptr(t) for t in L]) for L in (Qs, Ks, Vs, Os)]
    check(lib().tl_sp_attention_loopback(comm._h, *[a[0] for a in arrs], S_r * comm.world, heads, D, scale,
                                         _stream(stream)), "tl_sp_attention_loopback")
    return Os


def static_map_device(M: int, world: int, tm_rows: int, channels_per_rank: int, n: int):
    """Device-evaluated static mapping rows (row_lo, row_hi, src_rank, channel) for tiles 0..n-1."""
    out = (C.c_int64 * (4 * n))()
    check(lib().tl_debug_static_map(M, world, tm_rows, channels_per_rank, n, out), "tl_debug_static_map")
    return [tuple(out[4 * i:4 * i + 4]) for i in range(n)]
