"""TEST INFRASTRUCTURE ONLY — ctypes access to the two CPU checkers.

* ``Restatement`` wraps ``oracle/_ref/liboracle.so``: our plain-C restatement
  of the reference's token-tree verification path (``oracle/restate.c``;
  every function cites the reference file:line it follows).
* ``Reference`` wraps ``oracle/_ref/libspectree_ref.so``: the UNMODIFIED
  reference (``/root/reference/proj/src/{token_tree,transformer,speculator,
  engine}.cpp``) compiled from its own sources by ``oracle/Makefile``, behind
  our C shim ``oracle/ref_shim.cpp``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module, and only
as the checker or the reported CPU baseline. The product package
(``paper_2305_09781_b200``) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_ip = C.POINTER(C.c_int)
_i64ptr = C.POINTER(C.c_int64)

# spectree::Errc order (proj/include/spectree/error.hpp:8-25)
ERRC = ["empty_input", "root_mismatch", "unknown_node", "missing_output", "tree_too_large",
        "tree_too_deep", "shape_mismatch", "prompt_too_long", "cache_gap", "chain_not_linked",
        "empty_context", "incomplete_profile", "bad_magic", "crc_mismatch", "io_error",
        "invalid_argument"]


class OracleError(RuntimeError):
    def __init__(self, status: int, what: str = ""):
        self.status = status
        self.code = ERRC[status - 1] if 0 < status <= len(ERRC) else f"status{status}"
        super().__init__(f"{self.code}: {what}")


def build(ref: bool = True) -> None:
    """Compile the checkers (restatement always; the reference when its sources exist)."""
    targets = ["restate"]
    if ref and os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def _flatten(seqs):
    lens = np.array([len(s) for s in seqs], dtype=np.int32)
    flat = np.array([t for s in seqs for t in s], dtype=np.int32) if len(seqs) else np.zeros(0, np.int32)
    if flat.size == 0:
        flat = np.zeros(1, np.int32)
    return flat, lens


class Restatement:
    def __init__(self, path: str | None = None):
        path = path or os.path.join(REF_DIR, "liboracle.so")
        if not os.path.exists(path):
            build(ref=False)
        L = self.lib = C.CDLL(path)
        L.or_merge.argtypes = [_i32p, _i32p, C.c_int, C.c_int, _i32p, _i32p, _i32p, C.c_int, _ip]
        L.or_verify.argtypes = [_i32p, _i32p, C.c_int, _i32p, C.c_int, _i32p, _i32p, _ip]
        L.or_argmax_f64.argtypes = [_f64p, C.c_int]
        L.or_argmax_f32.argtypes = [_f32p, C.c_int]
        L.or_ancestor_masks.argtypes = [_i32p, C.c_int, C.c_int, _u64p]
        L.or_uniform_stream.argtypes = [C.c_uint64, C.c_int64, C.c_double, C.c_double, _f64p]
        L.or_tree_attention.argtypes = [_f64p, _f64p, _f64p, _u64p, _i32p, _i32p, C.c_int, C.c_int,
                                        C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                        _f64p, C.c_void_p]
        L.or_greedy_verify.argtypes = [_f32p, C.c_int, _i32p, _i32p, C.c_int, _i32p, _i32p, _i32p, _ip]
        if hasattr(L, "or_mss_verify"):
            L.or_mss_verify.argtypes = [_f32p, _f32p, C.c_int, _i32p, _i32p, C.c_int, C.c_float,
                                        _f32p, C.c_int, _i32p, _i32p, _ip]

    def merge(self, seqs, max_nodes=64):
        flat, lens = _flatten(seqs)
        cap = int(lens.sum()) + 1 if len(seqs) else 1
        tok, par, dep = (np.zeros(cap, np.int32) for _ in range(3))
        n = C.c_int(0)
        st = self.lib.or_merge(flat, lens, len(seqs), max_nodes, tok, par, dep, cap, C.byref(n))
        if st != 0:
            raise OracleError(st, "merge")
        k = n.value
        return tok[:k].copy(), par[:k].copy(), dep[:k].copy()

    def verify(self, tok, par, outputs):
        tok = np.ascontiguousarray(tok, np.int32)
        par = np.ascontiguousarray(par, np.int32)
        outputs = np.ascontiguousarray(outputs, np.int32)
        n = len(tok)
        ver = np.zeros(n + 1, np.int32)
        ids = np.zeros(n + 1, np.int32)
        m = C.c_int(0)
        st = self.lib.or_verify(tok, par, n, outputs, len(outputs), ver, ids, C.byref(m))
        if st != 0:
            raise OracleError(st, "verify")
        return ver[: m.value].copy(), ids[: m.value].copy()

    def argmax(self, x):
        x = np.ascontiguousarray(x)
        if x.dtype == np.float64:
            return self.lib.or_argmax_f64(x, x.size)
        return self.lib.or_argmax_f32(np.ascontiguousarray(x, np.float32), x.size)

    def ancestor_masks(self, par, W=None):
        par = np.ascontiguousarray(par, np.int32)
        n = len(par)
        W = W or max(1, (n + 63) // 64)
        out = np.zeros(n * W, np.uint64)
        self.lib.or_ancestor_masks(par, n, W, out)
        return out.reshape(n, W)

    def uniform_stream(self, seed, n, lo, hi):
        out = np.zeros(n, np.float64)
        self.lib.or_uniform_stream(seed, n, lo, hi, out)
        return out

    def tree_attention(self, q, kc, vc, mask, P, n_nodes, scale, want_lse=False):
        """q [B,T,H,D]; kc/vc [B,Hkv,Lmax,D]; mask [B,T,W] u64 -> o [B,T,H,D] f64."""
        q = np.ascontiguousarray(q, np.float64)
        kc = np.ascontiguousarray(kc, np.float64)
        vc = np.ascontiguousarray(vc, np.float64)
        mask = np.ascontiguousarray(mask, np.uint64)
        B, T, H, D = q.shape
        Hkv, Lmax = kc.shape[1], kc.shape[2]
        W = mask.shape[-1]
        o = np.zeros_like(q)
        lse = np.zeros((B, H, T), np.float64) if want_lse else None
        self.lib.or_tree_attention(q, kc, vc, mask, np.ascontiguousarray(P, np.int32),
                                   np.ascontiguousarray(n_nodes, np.int32), B, T, H, Hkv, D, Lmax, W,
                                   float(scale), o,
                                   lse.ctypes.data_as(C.c_void_p) if want_lse else None)
        return (o, lse) if want_lse else o

    def greedy_verify(self, logits, tok, par):
        logits = np.ascontiguousarray(logits, np.float32)
        n, V = logits.shape
        outs = np.zeros(n, np.int32)
        ver = np.zeros(n + 1, np.int32)
        ids = np.zeros(n + 1, np.int32)
        m = C.c_int(0)
        st = self.lib.or_greedy_verify(logits, V, np.ascontiguousarray(tok, np.int32),
                                       np.ascontiguousarray(par, np.int32), n, outs, ver, ids,
                                       C.byref(m))
        if st != 0:
            raise OracleError(st, "greedy_verify")
        return outs, ver[: m.value].copy(), ids[: m.value].copy()

    def mss_verify(self, logits, q, tok, par, temperature, uniforms):
        logits = np.ascontiguousarray(logits, np.float32)
        q = np.ascontiguousarray(q, np.float32)
        n, V = logits.shape
        u = np.ascontiguousarray(uniforms, np.float32)
        ver = np.zeros(n + 1, np.int32)
        ids = np.zeros(n + 1, np.int32)
        m = C.c_int(0)
        st = self.lib.or_mss_verify(logits, q, V, np.ascontiguousarray(tok, np.int32),
                                    np.ascontiguousarray(par, np.int32), n, float(temperature), u,
                                    len(u), ver, ids, C.byref(m))
        if st != 0:
            raise OracleError(st, "mss_verify")
        return ver[: m.value].copy(), ids[: m.value].copy()


class Reference:
    """The unmodified reference library (oracle/_ref/libspectree_ref.so)."""

    def __init__(self, path: str | None = None):
        path = path or os.path.join(REF_DIR, "libspectree_ref.so")
        if not os.path.exists(path):
            build(ref=True)
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_merge.argtypes = [_i32p, _i32p, C.c_int, C.c_int, _i32p, _i32p, _i32p, C.c_int, _ip]
        L.ref_dfs_chains.argtypes = [_i32p, _i32p, C.c_int, C.c_int, _i32p, _i32p, C.c_int, _ip]
        L.ref_verify.argtypes = [_i32p, _i32p, C.c_int, C.c_int, _i32p, C.c_int, _i32p, C.c_int, _ip]
        L.ref_argmax.argtypes = [_f64p, C.c_int]
        L.ref_attention.argtypes = [_f64p] * 5 + [C.c_int, C.c_int, C.c_int, _f64p, _f64p]
        cfg = [C.c_int] * 6
        L.ref_param_count.argtypes = cfg
        L.ref_param_count.restype = C.c_int64
        L.ref_init_weights.argtypes = cfg + [C.c_uint64, _f64p, C.c_int64]
        L.ref_tree_decode.argtypes = cfg + [C.c_uint64, _i32p, C.c_int, _i32p, _i32p, C.c_int,
                                            C.c_int, C.c_int, _f64p, _i32p, C.c_int, _ip]
        L.ref_per_path_logits.argtypes = cfg + [C.c_uint64, _i32p, C.c_int, _i32p, C.c_int, _f64p]
        L.ref_run_incremental.argtypes = cfg + [C.c_uint64, _i32p, C.c_int, C.c_int, C.c_int32,
                                                _i32p, C.c_int, _ip, _i64ptr]
        L.ref_run_speculative_self.argtypes = cfg + [C.c_uint64, _i32p, C.c_int, C.c_int, C.c_int32,
                                                     C.c_int, C.c_int, C.c_int, _i32p, C.c_int, _ip,
                                                     _i64ptr]
        L.ref_bench_tree_decode.argtypes = cfg + [C.c_uint64, C.c_int, C.c_int, _i32p, _i32p,
                                                  C.c_int, C.c_int, C.c_int]
        L.ref_bench_tree_decode.restype = C.c_double
        L.ref_beam_speculate.argtypes = cfg + [C.c_uint64, _i32p, C.c_int, C.c_int, C.c_int,
                                               C.c_int32, _i32p, _i32p, C.c_int, _ip]
        L.ref_next_log_probs.argtypes = cfg + [C.c_uint64, _i32p, C.c_int, _f64p]

    def _check(self, st, what):
        if st != 0:
            raise OracleError(st, f"{what}: {self.lib.ref_last_error().decode()}")

    def merge(self, seqs, max_nodes=64):
        flat, lens = _flatten(seqs)
        cap = int(lens.sum()) + 1 if len(seqs) else 1
        tok, par, dep = (np.zeros(cap, np.int32) for _ in range(3))
        n = C.c_int(0)
        self._check(self.lib.ref_merge(flat, lens, len(seqs), max_nodes, tok, par, dep, cap,
                                       C.byref(n)), "merge")
        k = n.value
        return tok[:k].copy(), par[:k].copy(), dep[:k].copy()

    def dfs_chains(self, seqs, max_nodes=64):
        flat, lens = _flatten(seqs)
        cap = int(lens.sum()) + 1
        ids = np.zeros(cap, np.int32)
        clen = np.zeros(cap, np.int32)
        n = C.c_int(0)
        self._check(self.lib.ref_dfs_chains(flat, lens, len(seqs), max_nodes, ids, clen, cap,
                                            C.byref(n)), "dfs_chains")
        out, at = [], 0
        for c in range(n.value):
            out.append(ids[at: at + clen[c]].tolist())
            at += clen[c]
        return out

    def verify(self, seqs, outputs, max_nodes=64):
        flat, lens = _flatten(seqs)
        outputs = np.ascontiguousarray(outputs, np.int32)
        cap = len(outputs) + 2
        ver = np.zeros(cap, np.int32)
        n = C.c_int(0)
        self._check(self.lib.ref_verify(flat, lens, len(seqs), max_nodes, outputs,
                                        len(outputs), ver, cap, C.byref(n)), "verify")
        return ver[: n.value].copy()

    def attention(self, x, wq, wk, wv, wo, heads, mask):
        x = np.ascontiguousarray(x, np.float64)
        l, d = x.shape
        out = np.zeros((l, d), np.float64)
        f = lambda a: np.ascontiguousarray(a, np.float64)  # noqa: E731
        self._check(self.lib.ref_attention(x, f(wq), f(wk), f(wv), f(wo), l, d, heads, f(mask),
                                           out), "attention")
        return out

    def init_weights(self, cfg, seed):
        n = self.lib.ref_param_count(*cfg)
        out = np.zeros(n, np.float64)
        self._check(self.lib.ref_init_weights(*cfg, seed, out, n), "init_weights")
        return out

    def tree_decode(self, cfg, seed, prompt, seqs, max_nodes=64, apply_fix=True):
        flat, lens = _flatten(seqs)
        prompt = np.ascontiguousarray(prompt, np.int32)
        cap = int(lens.sum()) + 1
        V = cfg[3]
        logits = np.zeros(cap * V, np.float64)
        toks = np.zeros(cap, np.int32)
        n = C.c_int(0)
        self._check(self.lib.ref_tree_decode(*cfg, seed, prompt, len(prompt), flat, lens,
                                             len(seqs), max_nodes, int(apply_fix), logits, toks,
                                             cap, C.byref(n)), "tree_decode")
        k = n.value
        return logits[: k * V].reshape(k, V).copy(), toks[:k].copy()

    def per_path_logits(self, cfg, seed, prompt, path):
        prompt = np.ascontiguousarray(prompt, np.int32)
        plen = len(path)
        path = np.ascontiguousarray(path, np.int32) if plen else np.zeros(1, np.int32)
        out = np.zeros(cfg[3], np.float64)
        self._check(self.lib.ref_per_path_logits(*cfg, seed, prompt, len(prompt), path, plen, out),
                    "per_path_logits")
        return out

    def run_incremental(self, cfg, seed, prompt, max_new, eos=-1):
        prompt = np.ascontiguousarray(prompt, np.int32)
        cap = len(prompt) + max_new + 1
        seq = np.zeros(cap, np.int32)
        n = C.c_int(0)
        steps = C.c_int64(0)
        self._check(self.lib.ref_run_incremental(*cfg, seed, prompt, len(prompt), max_new, eos,
                                                 seq, cap, C.byref(n), C.byref(steps)),
                    "run_incremental")
        return seq[: n.value].copy(), steps.value

    def run_speculative_self(self, cfg, seed, prompt, max_new, beam_width, beam_depth, eos=-1,
                             max_tree_nodes=64):
        prompt = np.ascontiguousarray(prompt, np.int32)
        cap = len(prompt) + max_new + 1
        seq = np.zeros(cap, np.int32)
        n = C.c_int(0)
        steps = C.c_int64(0)
        self._check(self.lib.ref_run_speculative_self(*cfg, seed, prompt, len(prompt), max_new,
                                                      eos, beam_width, beam_depth, max_tree_nodes,
                                                      seq, cap, C.byref(n), C.byref(steps)),
                    "run_speculative")
        return seq[: n.value].copy(), steps.value

    def beam_speculate(self, cfg, seed, prefix, width, depth, eos=-1):
        prefix = np.ascontiguousarray(prefix, np.int32)
        cap = (len(prefix) + depth + 1) * width + 1
        flat = np.zeros(cap, np.int32)
        lens = np.zeros(width + 1, np.int32)
        n = C.c_int(0)
        self._check(self.lib.ref_beam_speculate(*cfg, seed, prefix, len(prefix), width, depth, eos,
                                                flat, lens, cap, C.byref(n)), "beam_speculate")
        out, at = [], 0
        for i in range(n.value):
            out.append(flat[at: at + lens[i]].tolist())
            at += lens[i]
        return out

    def next_log_probs(self, cfg, seed, ctx):
        ctx = np.ascontiguousarray(ctx, np.int32)
        out = np.zeros(cfg[3], np.float64)
        self._check(self.lib.ref_next_log_probs(*cfg, seed, ctx, len(ctx), out), "next_log_probs")
        return out

    def bench_tree_decode(self, cfg, seed, n_requests, prefix_len, seqs, max_nodes, n_threads):
        flat, lens = _flatten(seqs)
        s = self.lib.ref_bench_tree_decode(*cfg, seed, n_requests, prefix_len, flat, lens,
                                           len(seqs), max_nodes, n_threads)
        if s < 0:
            raise OracleError(int(-s), self.lib.ref_last_error().decode())
        return s


def available_reference() -> bool:
    return os.path.exists(os.path.join(REF_DIR, "libspectree_ref.so"))
