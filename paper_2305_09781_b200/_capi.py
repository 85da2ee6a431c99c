"""ctypes binding of the C-ABI (include/spectree_capi.h) over torch tensors.

torch is only plumbing here (device memory and streams); every computation
goes through ``libspectree_b200.so``. There is no CPU fallback: if the library
or a CUDA device is missing, calls raise ``SpectreeError``.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libspectree_b200.so")

# 1 + spectree::Errc (reference proj/include/spectree/error.hpp:8-25)
ERRC = ["empty_input", "root_mismatch", "unknown_node", "missing_output", "tree_too_large",
        "tree_too_deep", "shape_mismatch", "prompt_too_long", "cache_gap", "chain_not_linked",
        "empty_context", "incomplete_profile", "bad_magic", "crc_mismatch", "io_error",
        "invalid_argument"]
EXTRA = {100: "no_device", 101: "cuda_error", 102: "unsupported"}

DTYPES = {torch.float16: 0, torch.bfloat16: 1, torch.float32: 2, torch.float64: 3}


class SpectreeError(RuntimeError):
    """Mirror of spectree::Error: carries the Errc name in ``.code``."""

    def __init__(self, status: int, msg: str):
        self.status = status
        self.code = ERRC[status - 1] if 0 < status <= len(ERRC) else EXTRA.get(status, str(status))
        super().__init__(f"[{self.code}] {msg}")


class PeerOut(C.Structure):
    _fields_ = [("world", C.c_int), ("rank", C.c_int), ("out", C.c_void_p)]


class AttnArgs(C.Structure):
    _fields_ = [("dtype", C.c_int), ("B", C.c_int), ("T", C.c_int), ("H", C.c_int),
                ("Hkv", C.c_int), ("D", C.c_int), ("W", C.c_int), ("Lmax", C.c_int64),
                ("q", C.c_void_p), ("k_cache", C.c_void_p), ("v_cache", C.c_void_p),
                ("mask", C.c_void_p), ("prefix_len", C.c_void_p), ("n_nodes", C.c_void_p),
                ("o", C.c_void_p), ("lse", C.c_void_p), ("scale", C.c_double),
                ("workspace", C.c_void_p), ("workspace_bytes", C.c_size_t),
                ("force_path", C.c_int), ("k_tree", C.c_void_p), ("v_tree", C.c_void_p),
                ("early_kv", C.c_int), ("q_rows", C.c_int), ("q_node0", C.c_int)]


_lib = None

# every exported symbol and its signature (restype, argtypes)
_V, _I, _I64, _Z, _D, _F = C.c_void_p, C.c_int, C.c_int64, C.c_size_t, C.c_double, C.c_float
SIGNATURES = {
    "st_abi_version": (_I, []),
    "st_last_error_message": (C.c_char_p, []),
    "st_device_count": (_I, []),
    "st_tree_attention_workspace_size": (_Z, [C.POINTER(AttnArgs)]),
    "st_tree_attention": (_I, [C.POINTER(AttnArgs), _V]),
    "st_tree_attention_path": (_I, [C.POINTER(AttnArgs)]),
    "st_kv_append": (_I, [_I, _I, _I, _I, _I, _I64, _V, _V, _V, _V, _V, _V, _V]),
    "st_kv_compact": (_I, [_I, _I, _I, _I, _I64, _I, _I64, _V, _I, _V, _V, _V, _V, _V, _V]),
    "st_tree_prepare": (_I, [_I, _I, _I, _I, _I, _I64, _V, _V, _V, _V, _V, _V, _V, _I, _V, _V]),
    "st_heads_gather_layout": (_I, [_I, _I, _I, _I, _I, _I, _V, _V, _V]),
    "st_verify_workspace_size": (_Z, [_I, _I]),
    "st_verify_greedy": (_I, [_V, _I, _I, _I, _V, _V, _V, _V, C.c_int32, _V, _V, _V, _V, _V, _V]),
    "st_verify_greedy_compact": (_I, [_V, _I, _I, _I, _V, _V, _V, _V, C.c_int32, _V, _V, _V, _V, _V,
                                      _I, _I, _I, _I64, _I, _I64, _V, _V, _V, _V, _I64, _V, _V,
                                      _V]),
    "st_verify_outputs": (_I, [_V, _I, _I, _V, _V, _V, _V, C.c_int32, _V, _V, _V, _V]),
    "st_verify_mss": (_I, [_V, _V, _I, _I, _I, _V, _V, _V, _F, _V, _I, _V, _V, _V, _V]),
    "st_build_masks": (_I, [_V, _V, _I, _I, _I, _V, _V]),
    "st_build_masks_early": (_I, [_V, _V, _I, _I, _I, _V, _V]),
    "st_model_create": (_I, [_V, C.c_uint64, _I, _V]),
    "st_model_destroy": (None, [_V]),
    "st_model_param_count": (_Z, [_V]),
    "st_model_workspace_size": (_Z, [_V, _I, _I]),
    "st_model_tree_forward": (_I, [_V, _I, _I, _V, _V, _V, _I, _V, _V, _V, _V, _I64, _V, _V, _Z, _V]),
    "st_tree_merge": (_I, [_V, _V, _I, _I, _V, _V, _V, _I, C.POINTER(_I)]),
    "st_tree_merge_batch": (_I, [_I, _V, _V, _V, _I, _I, _V, _V, _V, _V, _V, _I]),
    "st_tree_attention_allgather": (_I, [C.POINTER(AttnArgs), C.POINTER(PeerOut), _V]),
    "st_peer_signal": (_I, [_V, _I, _I, C.c_uint32, _V]),
    "st_peer_wait": (_I, [_V, _I, C.c_uint32, _V]),
    "st_model_get_config": (None, [_V, _V]),
    "st_model_get_dtype": (_I, [_V]),
    "st_engine_create": (_I, [_V, _V, _V, _V]),
    "st_engine_destroy": (None, [_V]),
    "st_engine_tree_nodes": (_I, [_V]),
    "st_engine_start": (_I, [_V, _I, _V, _V, _V, _V]),
    "st_engine_step": (_I, [_V, _V]),
    "st_engine_read": (_I, [_V, _V, _V, _V, _V]),
    "st_engine_sequence": (_I, [_V, _I, _V, _I, C.POINTER(_I), _V]),
    "st_comm_get_unique_id": (_I, [_V]),
    "st_comm_init": (_I, [_I, _I, _V, _V]),
    "st_comm_allgather": (_I, [_V, _V, _V, _Z, _V]),
    "st_comm_gather_accepted": (_I, [_V, _V, _V, _I, _I, _V, _V, _V]),
    "st_comm_size": (_I, [_V]),
    "st_comm_rank": (_I, [_V]),
    "st_comm_destroy": (None, [_V]),
    "st_verify_plan_create": (_I, [_V, _V]),
    "st_verify_plan_run": (_I, [_V, _V]),
    "st_verify_plan_destroy": (None, [_V]),
    "st_kv_commit_tree": (_I, [_I, _I, _I, _I, _I, _I64, _I, _I64, _V, _I, _V, _V, _V, _V, _V,
                               _I64, _V, _V, _V]),
    "st_model_tree_forward_kt": (_I, [_V, _I, _I, _V, _V, _V, _I, _V, _V, _V, _V, _I64, _V, _V,
                                      _V, _Z, _V]),
    "st_model_tree_forward_slice": (_I, [_V, _I, _I, _I, _I, _V, _V, _V, _I, _V, _V, _V, _V,
                                         _I64, _V, _V, _V, _Z, _V]),
    "st_gemm": (_I, [_I, _I, _I, _I, _I, _V, _I, _V, _I, _V, _I, _I64, _I, _V]),
}


def lib():
    """Load libspectree_b200.so (fails loudly: no fallback exists)."""
    global _lib
    if _lib is None:
        # ST_LIB_VARIANT (diagnostic A/B runs only): an alternative build of the
        # same library, e.g. build/variants/<name>.so
        path = os.environ.get("ST_LIB_VARIANT") or _LIB_PATH
        if not os.path.exists(path):
            raise SpectreeError(102, f"{path} missing: run __graft_entry__.build()")
        L = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            if hasattr(L, name):
                fn = getattr(L, name)
                fn.restype, fn.argtypes = res, args
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != 0:
        raise SpectreeError(status, lib().st_last_error_message().decode())


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


# ------------------------------------------------------------------ K1 ----
def attn_args(q, k_cache, v_cache, mask, prefix_len, n_nodes, out, lse=None, scale=None,
              workspace=None, force_path=0, k_tree=None, v_tree=None, early_kv=False,
              q_node0=None):
    B, T, H, D = q.shape
    q_rows = 0
    if q_node0 is not None:   # q holds nodes [q_node0, q_node0 + q.shape[1]) of T = mask rows
        q_rows, T = q.shape[1], mask.shape[1]
    Hkv, Lmax = k_cache.shape[1], k_cache.shape[2]
    a = AttnArgs()
    a.dtype = DTYPES[q.dtype]
    a.B, a.T, a.H, a.Hkv, a.D, a.W, a.Lmax = B, T, H, Hkv, D, mask.shape[-1], Lmax
    a.q, a.k_cache, a.v_cache = q.data_ptr(), k_cache.data_ptr(), v_cache.data_ptr()
    a.mask, a.prefix_len, a.n_nodes = mask.data_ptr(), prefix_len.data_ptr(), n_nodes.data_ptr()
    a.o = out.data_ptr() if out is not None else None
    a.lse = lse.data_ptr() if lse is not None else None
    a.scale = float(scale if scale is not None else D ** -0.5)
    a.workspace = workspace.data_ptr() if workspace is not None else None
    a.workspace_bytes = workspace.numel() if workspace is not None else 0
    a.force_path = force_path
    a.k_tree = k_tree.data_ptr() if k_tree is not None else None
    a.v_tree = v_tree.data_ptr() if v_tree is not None else None
    a.early_kv = 1 if early_kv else 0
    a.q_rows = q_rows
    a.q_node0 = int(q_node0) if q_node0 is not None else 0
    return a


def tree_attention_workspace(q, k_cache, v_cache, mask, prefix_len, n_nodes, force_path=0):
    out = torch.empty_like(q)
    a = attn_args(q, k_cache, v_cache, mask, prefix_len, n_nodes, out, force_path=force_path)
    n = lib().st_tree_attention_workspace_size(C.byref(a))
    return torch.zeros(max(int(n), 1), dtype=torch.uint8, device=q.device)


def tree_attention_path(q, k_cache, v_cache, mask, prefix_len, n_nodes, force_path=0):
    out = torch.empty_like(q)
    a = attn_args(q, k_cache, v_cache, mask, prefix_len, n_nodes, out, force_path=force_path)
    return int(lib().st_tree_attention_path(C.byref(a)))


def tree_attention(q, k_cache, v_cache, mask, prefix_len, n_nodes, out=None, lse=None,
                   scale=None, workspace=None, force_path=0, stream=None, k_tree=None,
                   v_tree=None, early_kv=False, q_node0=None):
    """K1 through st_tree_attention. Shapes: q [B,T,H,D]; caches [B,Hkv,Lmax,D];
    mask [B,T,W] int64 (uint64 bits); prefix_len/n_nodes [B] int32 (device);
    k_tree/v_tree (optional) [B,T,Hkv,D]: the tree rows, read instead of cache
    rows [P, P+n). q_node0 (tcgen05 path: needs k_tree): q / out / lse hold only the nodes
    [q_node0, q_node0 + q.shape[1]) of the T = mask.shape[1] tree nodes."""
    if out is None:
        out = torch.empty_like(q)
    if workspace is None:
        workspace = tree_attention_workspace(q, k_cache, v_cache, mask, prefix_len, n_nodes,
                                             force_path)
    a = attn_args(q, k_cache, v_cache, mask, prefix_len, n_nodes, out, lse, scale, workspace,
                  force_path, k_tree, v_tree, early_kv, q_node0)
    check(lib().st_tree_attention(C.byref(a), _stream(stream)))
    return out


def tree_attention_allgather(q, k_cache, v_cache, mask, prefix_len, n_nodes, out_ptrs, world,
                             rank, lse=None, scale=None, workspace=None, stream=None):
    """Head-sharded K1 with the all-gather fused into the epilogue
    (st_tree_attention_allgather): this rank's heads q [B,T,H,D] are written
    into every rank's [B,T,world*H,D] buffer; out_ptrs is a device int64
    tensor [world] of (peer-mapped) buffer addresses."""
    assert out_ptrs.dtype == torch.int64 and out_ptrs.is_cuda and out_ptrs.numel() == world
    if workspace is None:
        workspace = tree_attention_workspace(q, k_cache, v_cache, mask, prefix_len, n_nodes)
    a = attn_args(q, k_cache, v_cache, mask, prefix_len, n_nodes, None, lse, scale, workspace, 0)
    po = PeerOut(int(world), int(rank), out_ptrs.data_ptr())
    check(lib().st_tree_attention_allgather(C.byref(a), C.byref(po), _stream(stream)))


def peer_signal(signal_ptrs, world, rank, epoch, stream=None):
    """Publish `epoch` into slot `rank` of every rank's signal array
    (signal_ptrs: device int64 tensor [world] of peer-mapped uint32[world])."""
    check(lib().st_peer_signal(C.c_void_p(signal_ptrs.data_ptr()), int(world), int(rank),
                               int(epoch) & 0xFFFFFFFF, _stream(stream)))


def peer_wait(my_signals, world, epoch, stream=None):
    """Hold the stream until every slot of my_signals (int32 [world]) reached epoch."""
    check(lib().st_peer_wait(_ptr(my_signals), int(world), int(epoch) & 0xFFFFFFFF,
                             _stream(stream)))


# ------------------------------------------------------------------ K2 ----
def kv_append(k_new, v_new, prefix_len, n_nodes, k_cache, v_cache, stream=None):
    B, T, Hkv, D = k_new.shape
    check(lib().st_kv_append(DTYPES[k_new.dtype], B, T, Hkv, D, k_cache.shape[-2], _ptr(k_new),
                             _ptr(v_new), _ptr(prefix_len), _ptr(n_nodes), _ptr(k_cache),
                             _ptr(v_cache), _stream(stream)))


def tree_prepare(k_new, v_new, prefix_len, n_nodes, k_cache, v_cache, parent, W=None, out=None,
                 stream=None):
    """K2 append + ancestor masks in one launch; returns the [B, T, W] int64 masks."""
    B, T, Hkv, D = k_new.shape
    W = W or (T + 63) // 64
    mask = out if out is not None else torch.empty((B, T, W), dtype=torch.int64, device=k_new.device)
    check(lib().st_tree_prepare(DTYPES[k_new.dtype], B, T, Hkv, D, k_cache.shape[-2], _ptr(k_new),
                                _ptr(v_new), _ptr(prefix_len), _ptr(n_nodes), _ptr(k_cache),
                                _ptr(v_cache), _ptr(parent), W, _ptr(mask), _stream(stream)))
    return mask


def kv_compact(ids, n_keep, prefix_len, k_cache, v_cache, new_prefix_len=None, stream=None):
    """k_cache/v_cache: [L,B,Hkv,Lmax,D] (layer-major) or [B,Hkv,Lmax,D]."""
    if k_cache.dim() == 4:
        n_layers, layer_stride = 1, k_cache.numel()
        B, Hkv, Lmax, D = k_cache.shape
    else:
        n_layers = k_cache.shape[0]
        layer_stride = k_cache[0].numel()
        B, Hkv, Lmax, D = k_cache.shape[1:]
    check(lib().st_kv_compact(DTYPES[k_cache.dtype], B, Hkv, D, Lmax, n_layers, layer_stride,
                              _ptr(ids), ids.shape[-1], _ptr(n_keep), _ptr(prefix_len),
                              _ptr(new_prefix_len), _ptr(k_cache), _ptr(v_cache),
                              _stream(stream)))


def kv_commit_tree(ids, n_keep, prefix_len, tree_qkv, k_cache, v_cache, T, new_prefix_len=None,
                   stream=None):
    """Commit the accepted rows of every layer from tree_qkv
    ([L][3][B*T][d], DeviceModel.new_tree_qkv) into the caches [L][B][H][Lmax][D]."""
    n_layers, B, Hkv, Lmax, D = k_cache.shape
    rows = tree_qkv.shape[2]
    assert rows == B * T
    k_tree = tree_qkv[0, 1]
    v_tree = tree_qkv[0, 2]
    check(lib().st_kv_commit_tree(DTYPES[k_cache.dtype], B, T, Hkv, D, Lmax, n_layers,
                                  k_cache[0].numel(), _ptr(ids), ids.shape[-1], _ptr(n_keep),
                                  _ptr(prefix_len), _ptr(new_prefix_len), _ptr(k_tree),
                                  _ptr(v_tree), tree_qkv[0].numel(), _ptr(k_cache), _ptr(v_cache),
                                  _stream(stream)))


def heads_gather_layout(gathered, world, out=None, stream=None):
    """[world, B, T, Hl, D] -> [B, T, world*Hl, D] (C4 head-sharded outputs)."""
    W, B, T, Hl, D = gathered.shape
    assert W == world
    if out is None:
        out = torch.empty((B, T, world * Hl, D), dtype=gathered.dtype, device=gathered.device)
    check(lib().st_heads_gather_layout(DTYPES[gathered.dtype], world, B, T, Hl, D, _ptr(gathered),
                                       _ptr(out), _stream(stream)))
    return out


# ------------------------------------------------------------------ K3 ----
def verify_workspace(B, T, device="cuda"):
    n = lib().st_verify_workspace_size(B, T)
    return torch.zeros(int(n), dtype=torch.uint8, device=device)


def verify_greedy(logits, tokens, parent, n_nodes, budget=None, eos=-1, workspace=None,
                  stream=None, want_argmax=True, out=None):
    """out: optional preallocated (verified [B,T+1], ids [B,T+1], len [B]) int32."""
    B, T, V = logits.shape
    dev = logits.device
    argmax = torch.empty((B, T), dtype=torch.int32, device=dev) if want_argmax else None
    if out is None:
        verified = torch.full((B, T + 1), -1, dtype=torch.int32, device=dev)
        ids = torch.full((B, T + 1), -1, dtype=torch.int32, device=dev)
        length = torch.zeros(B, dtype=torch.int32, device=dev)
    else:
        verified, ids, length = out
    if workspace is None:
        workspace = verify_workspace(B, T, dev)
    check(lib().st_verify_greedy(_ptr(logits), B, T, V, _ptr(tokens), _ptr(parent), _ptr(n_nodes),
                                 _ptr(budget), int(eos), _ptr(argmax), _ptr(verified), _ptr(ids),
                                 _ptr(length), _ptr(workspace), _stream(stream)))
    return argmax, verified, ids, length


def verify_greedy_compact(logits, tokens, parent, n_nodes, prefix_len, k_cache, v_cache,
                          budget=None, eos=-1, workspace=None, new_prefix_len=None, stream=None,
                          want_argmax=True, out=None, k_tree=None, v_tree=None):
    """verify_greedy + kv_compact(ids, len) in two launches (walk fused into the
    compaction). k_cache/v_cache: [L,B,Hkv,Lmax,D] or [B,Hkv,Lmax,D].
    k_tree/v_tree ([L,]B,T,Hkv,D): copy the accepted rows from the tree's own
    K/V instead of moving them inside the cache (K1's k_tree mode)."""
    B, T, V = logits.shape
    dev = logits.device
    argmax = torch.empty((B, T), dtype=torch.int32, device=dev) if want_argmax else None
    if out is None:
        verified = torch.full((B, T + 1), -1, dtype=torch.int32, device=dev)
        ids = torch.full((B, T + 1), -1, dtype=torch.int32, device=dev)
        length = torch.zeros(B, dtype=torch.int32, device=dev)
    else:
        verified, ids, length = out
    if workspace is None:
        workspace = verify_workspace(B, T, dev)
    if k_cache.dim() == 4:
        n_layers, layer_stride = 1, k_cache.numel()
        _, Hkv, Lmax, D = k_cache.shape
    else:
        n_layers, layer_stride = k_cache.shape[0], k_cache[0].numel()
        _, Hkv, Lmax, D = k_cache.shape[1:]
    check(lib().st_verify_greedy_compact(
        _ptr(logits), B, T, V, _ptr(tokens), _ptr(parent), _ptr(n_nodes), _ptr(budget), int(eos),
        _ptr(argmax), _ptr(verified), _ptr(ids), _ptr(length), _ptr(workspace),
        DTYPES[k_cache.dtype], Hkv, D, Lmax, n_layers, layer_stride, _ptr(prefix_len),
        _ptr(new_prefix_len), _ptr(k_tree), _ptr(v_tree),
        (k_tree[0].numel() if k_tree is not None and k_tree.dim() == 5 else 0),
        _ptr(k_cache), _ptr(v_cache), _stream(stream)))
    return argmax, verified, ids, length


# ------------------------------------------------------------------ K4 ----
def verify_mss(logits, q, tokens, parent, n_nodes, temperature, uniforms, stream=None):
    B, T, V = logits.shape
    dev = logits.device
    verified = torch.full((B, T + 1), -1, dtype=torch.int32, device=dev)
    ids = torch.full((B, T + 1), -1, dtype=torch.int32, device=dev)
    length = torch.zeros(B, dtype=torch.int32, device=dev)
    check(lib().st_verify_mss(_ptr(logits), _ptr(q), B, T, V, _ptr(tokens), _ptr(parent),
                              _ptr(n_nodes), float(temperature), _ptr(uniforms),
                              uniforms.shape[-1], _ptr(verified), _ptr(ids), _ptr(length),
                              _stream(stream)))
    return verified, ids, length


# ---------------------------------------------------------------- masks ----
def build_masks(parent, n_nodes, W=None, stream=None, out=None, early=False):
    """Ancestor masks [B, T, W] int64. early=True: st_build_masks_early (the
    previous kernel on the stream neither writes parent/n_nodes nor touches
    the mask buffer)."""
    B, T = parent.shape
    W = W or (T + 63) // 64
    mask = out if out is not None else torch.empty((B, T, W), dtype=torch.int64,
                                                   device=parent.device)
    fn = lib().st_build_masks_early if early else lib().st_build_masks
    check(fn(_ptr(parent), _ptr(n_nodes), B, T, W, _ptr(mask), _stream(stream)))
    return mask


# ------------------------------------------------------ device model ----
class ModelConfig(C.Structure):
    _fields_ = [("num_layers", C.c_int), ("num_heads", C.c_int), ("d_model", C.c_int),
                ("vocab_size", C.c_int), ("max_positions", C.c_int), ("ffn_mult", C.c_int)]


class DeviceModel:
    """The reference decoder resident on the GPU (f16/bf16), weights generated
    on device from UniformStream(seed) — st_model_* of the C-ABI."""

    def __init__(self, num_layers, num_heads, d_model, vocab_size, max_positions, ffn_mult=4,
                 seed=42, dtype=torch.float16):
        self.cfg = ModelConfig(num_layers, num_heads, d_model, vocab_size, max_positions, ffn_mult)
        self.dtype = dtype
        h = C.c_void_p()
        check(lib().st_model_create(C.byref(self.cfg), seed, DTYPES[dtype], C.byref(h)))
        self.handle = h
        self._ws = None

    def __del__(self):
        if getattr(self, "handle", None):
            try:
                lib().st_model_destroy(self.handle)
            except TypeError:   # interpreter shutdown: module globals already cleared
                pass
            self.handle = None

    @property
    def param_count(self):
        return int(lib().st_model_param_count(self.handle))

    def new_cache(self, B, Lmax, device="cuda"):
        c = self.cfg
        shape = (c.num_layers, B, c.num_heads, Lmax, c.d_model // c.num_heads)
        return (torch.zeros(shape, dtype=self.dtype, device=device),
                torch.zeros(shape, dtype=self.dtype, device=device))

    def new_tree_qkv(self, B, T, device="cuda"):
        """[num_layers][3][B*T][d_model] buffer for tree_forward's k_tree mode."""
        c = self.cfg
        return torch.zeros((c.num_layers, 3, B * T, c.d_model), dtype=self.dtype, device=device)

    def tree_forward(self, tokens, positions, mask, prefix_len, n_nodes, k_cache, v_cache,
                     logits=None, stream=None, tree_qkv=None):
        """tree_qkv (optional, new_tree_qkv): K1's k_tree mode — the tree rows
        stay in tree_qkv (no per-layer append); commit with kv_commit_tree."""
        B, T = tokens.shape
        if logits is None:
            logits = torch.empty((B, T, self.cfg.vocab_size), dtype=torch.float32,
                                 device=tokens.device)
        need = int(lib().st_model_workspace_size(self.handle, B, T))
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.zeros(need, dtype=torch.uint8, device=tokens.device)
        if tree_qkv is None:
            check(lib().st_model_tree_forward(self.handle, B, T, _ptr(tokens), _ptr(positions),
                                              _ptr(mask), mask.shape[-1], _ptr(prefix_len),
                                              _ptr(n_nodes), _ptr(k_cache), _ptr(v_cache),
                                              k_cache.shape[-2], _ptr(logits), _ptr(self._ws),
                                              self._ws.numel(), _stream(stream)))
        else:
            check(lib().st_model_tree_forward_kt(self.handle, B, T, _ptr(tokens), _ptr(positions),
                                                 _ptr(mask), mask.shape[-1], _ptr(prefix_len),
                                                 _ptr(n_nodes), _ptr(k_cache), _ptr(v_cache),
                                                 k_cache.shape[-2], _ptr(tree_qkv), _ptr(logits),
                                                 _ptr(self._ws), self._ws.numel(),
                                                 _stream(stream)))
        return logits

    def tree_forward_slice(self, u0, nf, tokens, positions, mask, prefix_len, n_nodes, k_cache,
                           v_cache, tree_qkv, logits=None, stream=None):
        """st_model_tree_forward_slice: only nodes [u0, u0 + nf) of every
        request go through the model (one level of a tree grown level by
        level); their K/V land in tree_qkv, earlier slices' K/V are read from
        there. tokens / positions / mask are the full-tree arrays; n_nodes
        counts the nodes so far. logits (optional) [B, nf, V] f32."""
        B, T = tokens.shape
        need = int(lib().st_model_workspace_size(self.handle, B, T))
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.zeros(need, dtype=torch.uint8, device=tokens.device)
        check(lib().st_model_tree_forward_slice(
            self.handle, B, T, u0, nf, _ptr(tokens), _ptr(positions), _ptr(mask), mask.shape[-1],
            _ptr(prefix_len), _ptr(n_nodes), _ptr(k_cache), _ptr(v_cache), k_cache.shape[-2],
            _ptr(tree_qkv), _ptr(logits) if logits is not None else None, _ptr(self._ws),
            self._ws.numel(), _stream(stream)))
        return logits


# ------------------------------------------------------ device engine ----
class EngineConfig(C.Structure):
    _fields_ = [("max_batch", C.c_int), ("max_prompt", C.c_int), ("depth", C.c_int),
                ("expansion", C.c_int * 16), ("eos", C.c_int32)]


class Engine:
    """The device-resident speculative engine (st_engine_*): drafting with
    expansion trees on the GPU, LLM tree verification, greedy walk + commit
    with budgets / EOS on the device. ssm=None drafts with the LLM itself;
    expansion=() decodes one token per step."""

    def __init__(self, llm: DeviceModel, ssm: DeviceModel | None, max_batch: int, max_prompt: int,
                 expansion=(), eos: int = -1):
        cfg = EngineConfig()
        cfg.max_batch, cfg.max_prompt, cfg.depth, cfg.eos = max_batch, max_prompt, len(expansion), eos
        for i, e in enumerate(expansion):
            cfg.expansion[i] = int(e)
        h = C.c_void_p()
        check(lib().st_engine_create(llm.handle, ssm.handle if ssm is not None else None,
                                     C.byref(cfg), C.byref(h)))
        self.handle, self.llm, self.ssm, self.B = h, llm, ssm, max_batch
        self.T = int(lib().st_engine_tree_nodes(h))

    def __del__(self):
        if getattr(self, "handle", None):
            try:
                lib().st_engine_destroy(self.handle)
            except TypeError:   # interpreter shutdown
                pass
            self.handle = None

    def start(self, prompts, budgets, stream=None):
        import numpy as np
        flat = np.array([t for p in prompts for t in p], np.int32)
        lens = np.array([len(p) for p in prompts], np.int32)
        bud = np.array(budgets, np.int32)
        p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        check(lib().st_engine_start(self.handle, len(prompts), p(flat), p(lens), p(bud),
                                    _stream(stream)))

    def step(self, stream=None):
        check(lib().st_engine_step(self.handle, _stream(stream)))

    def read(self, stream=None):
        import numpy as np
        ver = np.zeros((self.B, self.T + 1), np.int32)
        ln = np.zeros(self.B, np.int32)
        done = np.zeros(self.B, np.int32)
        p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        check(lib().st_engine_read(self.handle, p(ver), p(ln), p(done), _stream(stream)))
        return ver, ln, done

    def sequence(self, b, stream=None):
        import numpy as np
        cap = 1 << 16
        out = np.zeros(cap, np.int32)
        n = C.c_int(0)
        check(lib().st_engine_sequence(self.handle, int(b), out.ctypes.data_as(C.c_void_p), cap,
                                       C.byref(n), _stream(stream)))
        return out[: n.value].tolist()

    def run(self, prompts, budgets, max_steps=100000, stream=None):
        """Generate until every request is done; returns (sequences, steps)."""
        self.start(prompts, budgets, stream)
        steps = 0
        while steps < max_steps:
            self.step(stream)
            steps += 1
            _, _, done = self.read(stream)
            if done[: len(prompts)].all():
                break
        return [self.sequence(b, stream) for b in range(len(prompts))], steps


# ------------------------------------------------------------ NCCL comm ----
class Comm:
    """st_comm_*: NCCL communicator of the C-ABI (DP exchange of accepted tokens)."""

    def __init__(self, nranks: int, rank: int, unique_id: bytes):
        assert len(unique_id) == 128
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        h = C.c_void_p()
        check(lib().st_comm_init(int(nranks), int(rank), buf, C.byref(h)))
        self.handle = h

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        check(lib().st_comm_get_unique_id(buf))
        return bytes(buf)

    def __del__(self):
        if getattr(self, "handle", None):
            try:
                lib().st_comm_destroy(self.handle)
            except TypeError:   # interpreter shutdown
                pass
            self.handle = None

    def gather_accepted(self, verified, length, pack, gathered, stream=None):
        B, T1 = verified.shape
        check(lib().st_comm_gather_accepted(self.handle, _ptr(verified), _ptr(length), B, T1 - 1,
                                            _ptr(pack), _ptr(gathered), _stream(stream)))
        return gathered


# ------------------------------------------------- verification step plan ----
class StepDesc(C.Structure):
    _fields_ = [("attn", AttnArgs), ("tokens", C.c_void_p), ("parent", C.c_void_p),
                ("logits", C.c_void_p), ("V", C.c_int), ("budget", C.c_void_p), ("eos", C.c_int32),
                ("verified", C.c_void_p), ("ids", C.c_void_p), ("len", C.c_void_p),
                ("verify_workspace", C.c_void_p), ("new_prefix_len", C.c_void_p),
                ("k_new", C.c_void_p), ("v_new", C.c_void_p)]


class VerifyPlan:
    """st_verify_plan_*: one verification step (masks -> K1 -> argmax -> walk +
    commit) prepared once and re-launched; consecutive runs chain with
    programmatic dependent launch. Holds references to every tensor it uses."""

    def __init__(self, q, k_cache, v_cache, mask, prefix_len, n_nodes, out, workspace, tokens,
                 parent, logits, verify_ws, verified, ids, length, k_tree=None, v_tree=None,
                 k_new=None, v_new=None, early_kv=True, budget=None, eos=-1, new_prefix_len=None):
        self._keep = [q, k_cache, v_cache, mask, prefix_len, n_nodes, out, workspace, tokens, parent,
                      logits, verify_ws, verified, ids, length, k_tree, v_tree, k_new, v_new,
                      budget, new_prefix_len]
        d = StepDesc()
        d.attn = attn_args(q, k_cache, v_cache, mask, prefix_len, n_nodes, out, workspace=workspace,
                           k_tree=k_tree, v_tree=v_tree, early_kv=early_kv)
        d.tokens, d.parent, d.logits = tokens.data_ptr(), parent.data_ptr(), logits.data_ptr()
        d.V = logits.shape[-1]
        d.budget = budget.data_ptr() if budget is not None else None
        d.eos = int(eos)
        d.verified, d.ids, d.len = verified.data_ptr(), ids.data_ptr(), length.data_ptr()
        d.verify_workspace = verify_ws.data_ptr()
        d.new_prefix_len = new_prefix_len.data_ptr() if new_prefix_len is not None else None
        d.k_new = k_new.data_ptr() if k_new is not None else None
        d.v_new = v_new.data_ptr() if v_new is not None else None
        h = C.c_void_p()
        check(lib().st_verify_plan_create(C.byref(d), C.byref(h)))
        self.handle = h
        self._run = lib().st_verify_plan_run

    def run(self, stream=None):
        st = self._run(self.handle, _stream(stream))
        if st != 0:
            check(st)

    def __del__(self):
        if getattr(self, "handle", None):
            try:
                lib().st_verify_plan_destroy(self.handle)
            except TypeError:   # interpreter shutdown
                pass
            self.handle = None


# ------------------------------------------------------------- GEMM ----
GEMM_EPI = {"store": 0, "gelu": 1, "add_to": 2, "store_f32": 3}


def gemm(a, w, out=None, epilogue="store", stream=None):
    """C (op)= A @ W on the tcgen05 GEMM (st_gemm). a [M][K]; w [K][N] or
    [Z][K][N]; out [M][N] / [Z][M][N] (f32 for epilogue="store_f32")."""
    M, K = a.shape
    Z = 1 if w.dim() == 2 else w.shape[0]
    N = w.shape[-1]
    if out is None:
        dt = torch.float32 if epilogue == "store_f32" else a.dtype
        out = torch.empty((M, N) if w.dim() == 2 else (Z, M, N), dtype=dt, device=a.device)
    check(lib().st_gemm(DTYPES[a.dtype], M, N, K, Z, _ptr(a), a.stride(0), _ptr(w), w.stride(-2),
                        _ptr(out),
                        out.stride(-2), (M * out.stride(-2)) if Z > 1 else 0, GEMM_EPI[epilogue],
                        _stream(stream)))
    return out
