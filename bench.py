#!/usr/bin/env python
"""Benchmark of the token-tree verification hot path (BASELINE.json metric:
"tree-verify tokens/s & KV HBM GB/s vs roofline at 1/2/4/8 B200; CPU ref
baseline").

Workload (config C2, BASELINE.json configs[1]): LLaMA-7B-shape attention layer,
fp16, batch 8 requests per GPU, 64-node token tree each, 2048 committed KV rows,
H = 32 heads x D = 128, greedy verification over a 32000-token vocabulary.

One step = one pass of the hot path over the batch (class VerifyStep, which
tests/test_gpu_step.py runs at the same shape against the oracle):
  ancestor bitmasks built on device
  -> K1 tree attention (tcgen05): committed KV from the cache, the tree's own
     K/V rows straight from their [B][T][H][D] tensors   [dominant kernel]
  -> K3 greedy verify (vocab argmax + accepted-path walk)
  -> K2 commit: the accepted path's K/V rows copied into the cache
  (+ N>1: NCCL all-gather of the accepted tokens — the DP exchange step, on a
     side stream, overlapping the next step)

value  = tree tokens verified per second over all ranks (B*T*N / step time),
         inputs resident in HBM, CUDA-event timed, max over ranks.
e2e    = same metric through the C-ABI with HOST buffers: every step copies
         Q, the tree's K/V and the tree topology from pinned host memory and
         reads the accepted tokens back (logits stay device-resident: in the
         full model they come from the on-device LM head).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                  [--config c2|c3|c4|c5] [--kv L] [--tree T]

--gpus N > 1 without a torchrun environment re-launches itself under
torch.distributed.run with N ranks (one GPU each, NCCL).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# C2
B, T, H, D, L, V = 8, 64, 32, 128, 2048, 32000
LAUNCHES_PER_STEP = 4          # masks, K1 (tree rows from k_tree), K3 argmax, K3 walk + K2 commit
STRONG_B_GLOBAL = 64           # strong-scaling companion: 64 requests split over the ranks
METRIC = "tree-verify tokens/s"
UNIT = "tokens/s"


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-strong", action="store_true",
                    help="skip the strong-scaling companion measurement")
    ap.add_argument("--tree-rows", default="own", choices=["own", "cache"],
                    help="K1 reads the tree rows from their own tensors (no append) or "
                         "from the cache after a K2 append")
    ap.add_argument("--config", default="c2", choices=["c2", "c3", "c4", "c5", "c3e"],
                    help="c2 (default, the headline metric); c3: full 32-layer 7B-shape stack, "
                         "batch 32 partitioned over the ranks, stochastic verification; c4: "
                         "LLaMA-65B-shape attention layer, heads sharded over the ranks; c5: "
                         "long-context verify step (B=16 per GPU, --kv, --tree); c3e: C3 model "
                         "shapes end to end through the device engine (st_engine: GPU drafting, "
                         "greedy tree verification, generation until every budget is spent)")
    ap.add_argument("--kv", type=int, default=32768, help="c5: committed KV rows")
    ap.add_argument("--tree", type=int, default=128, help="c5: tree nodes")
    ap.add_argument("--gather", default="nccl", choices=["nccl", "peer"],
                    help="c4: head-output all-gather through NCCL, or fused into K1's epilogue "
                         "over peer memory")
    return ap.parse_args(argv)


# ------------------------------------------------------------ launching ----
def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def maybe_spawn(args) -> bool:
    """--gpus N > 1 outside torchrun: re-launch this command under
    torch.distributed.run with N ranks. Returns True when it did (the parent
    then only relays the exit status)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return False
    env = dict(os.environ)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    r = subprocess.run(cmd, env=env)
    if r.returncode != 0:
        sys.exit(r.returncode)
    return True


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def dist_device(local):
    """GPU and process-group backend of this rank: NCCL, one GPU per rank.
    BENCH_SHARED_GPU_TEST=1 (code-path test only, numbers meaningless) lets N
    ranks share the visible GPUs over gloo, so the N>1 path runs on one GPU."""
    import torch
    if os.environ.get("BENCH_SHARED_GPU_TEST") == "1":
        return local % max(1, torch.cuda.device_count()), "gloo"
    return local, "nccl"


def init_rank(args):
    """Device + process group for this rank; fails loudly when the launch does
    not match --gpus (a silent 1-rank run would misreport n_gpus)."""
    import torch
    import torch.distributed as dist
    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (the product path has no CPU fallback)")
    local, backend = dist_device(local)
    if backend == "nccl" and local >= torch.cuda.device_count():
        raise SystemExit(f"bench.py: rank {rank} needs GPU {local}, only "
                         f"{torch.cuda.device_count()} visible")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":   # communicator-init lines (nranks) on stderr
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        dist.init_process_group(backend, device_id=dev if backend == "nccl" else None)
        t = torch.ones(1, device=dev)
        dist.all_reduce(t)
        assert int(t.item()) == world
        print(f"[bench] rank {rank}/{world}: {backend} communicator up, nranks={world}, "
              f"device cuda:{local}", file=sys.stderr, flush=True)
    return rank, world, local, dev


def finish_rank(world):
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


_ORIG_AFFINITY: set = set()


def bind_to_gpu_numa(local):
    """Pin this process to the host CPUs local to the GPU (sysfs local_cpulist),
    so pinned staging buffers are allocated on the GPU's NUMA node — what a
    serving deployment does. Returns the CPU count bound to (None if unknown)."""
    import torch
    try:
        pr = torch.cuda.get_device_properties(local)
        bus = "%04x:%02x:%02x.0" % (pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id)
        with open(f"/sys/bus/pci/devices/{bus}/local_cpulist") as f:
            spec = f.read().strip()
        cpus = set()
        for part in spec.split(","):
            lo, _, hi = part.partition("-")
            cpus.update(range(int(lo), int(hi or lo) + 1))
        cpus &= os.sched_getaffinity(0)
        if cpus:
            _ORIG_AFFINITY.update(os.sched_getaffinity(0))
            os.sched_setaffinity(0, cpus)
            return len(cpus)
    except (OSError, ValueError, AttributeError):
        pass
    return None


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def width_of(nodes):
    """SURVEY.md §8(d) tree construction: W root-to-leaf paths of depth
    ceil((T-1)/W): W=4 for T=16, 8 for T=64, 16 for T=128."""
    return max(1, min(16, nodes // 8))


def c2_trees(make_tree, seed, vocab, n_req=B, nodes=T):
    """W paths of depth ceil((T-1)/W) with uniform tokens, trimmed to exactly T nodes."""
    rng = np.random.default_rng(seed)
    width = width_of(nodes)
    depth = -(-(nodes - 1) // width)
    trees = []
    for _ in range(n_req):
        root = int(rng.integers(0, vocab))
        while True:
            seqs = [[root] + rng.integers(0, vocab, depth).tolist() for _ in range(width)]
            t = make_tree(seqs)
            # trim trailing tokens of the last paths until exactly `nodes`
            i = len(seqs) - 1
            while t.size > nodes and i >= 0:
                if len(seqs[i]) > 1:
                    seqs[i] = seqs[i][:-1]
                else:
                    i -= 1
                t = make_tree(seqs)
            if t.size == nodes:
                trees.append((t, seqs))
                break
    return trees


def c4_trees(make_tree, seed, n_req, vocab=V):
    """C4 trees: 3 SSMs, each expanded <1,1,3,1,1,1,1,1> (top-e_i children per
    frontier node at depth i), merged: 61 nodes."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n_req):
        root = int(rng.integers(0, vocab))
        seqs = []
        for _ssm in range(3):
            frontier = [[root]]
            for e in (1, 1, 3, 1, 1, 1, 1, 1):
                frontier = [p + [int(t)] for p in frontier for t in rng.integers(0, vocab, e)]
            seqs.extend(frontier)
        out.append((make_tree(seqs), seqs))
    return out


# ----------------------------------------------------------- the step ------
class VerifyStep:
    """One verification step over a batch, device-resident (C2 / C5 shapes).

    Buffers: KV cache [B][H][L+T][D] (fp16), Q and the tree's own K/V
    [B][T][H][D], logits [B][T][V] fp32 with planted acceptance (each node's
    argmax is its first child's token with probability 0.7), tree topology
    [B][T] int32. `run(a)` launches masks -> K1 -> K3 argmax -> K3 walk + K2
    commit on the current stream; `a` = (q, k_tree, v_tree, tokens, parents,
    n_nodes), so the e2e loop can swap in freshly copied inputs."""

    def __init__(self, dev, seed, B=B, T=T, L=L, H=H, D=D, V=V, tree_rows="own",
                 trees=None, dtype=None):
        import torch

        from paper_2305_09781_b200 import _capi
        from paper_2305_09781_b200.tree import TokenTree, TreeBatch
        self.capi = _capi
        self.B, self.T, self.L, self.H, self.D, self.V = B, T, L, H, D, V
        dtype = dtype or torch.float16
        if trees is None:
            trees = c2_trees(lambda s: TokenTree.merge_sequences(s, 1 << 20), 1000 + seed, V,
                             n_req=B, nodes=T)
        self.trees = trees
        self.batch = batch = TreeBatch([t for t, _ in trees], T)
        g = torch.Generator(device=dev).manual_seed(1234 + seed)
        Lmax = L + T
        self.kc = (torch.rand(B, H, Lmax, D, device=dev, generator=g) * 2 - 1).to(dtype)
        self.vc = (torch.rand(B, H, Lmax, D, device=dev, generator=g) * 2 - 1).to(dtype)
        self.q = (torch.rand(B, T, H, D, device=dev, generator=g) * 2 - 1).to(dtype)
        self.knew = (torch.rand(B, T, H, D, device=dev, generator=g) * 2 - 1).to(dtype)
        self.vnew = (torch.rand(B, T, H, D, device=dev, generator=g) * 2 - 1).to(dtype)
        self.logits = torch.randn(B, T, V, device=dev, generator=g)
        rng = np.random.default_rng(77 + seed)
        rows, cols = [], []
        for b in range(B):
            for u in range(batch.n_nodes[b]):
                kids = np.nonzero(batch.parents[b] == u)[0]
                if kids.size and rng.random() < 0.7:
                    rows.append(b * T + u)
                    cols.append(int(batch.tokens[b, kids[0]]))
        if rows:
            self.logits.view(B * T, V)[torch.tensor(rows, device=dev),
                                       torch.tensor(cols, device=dev)] = 50.0
        self.tok = torch.tensor(batch.tokens, device=dev)
        self.par = torch.tensor(batch.parents, device=dev)
        self.nn = torch.tensor(batch.n_nodes, device=dev)
        self.P = torch.full((B,), L, dtype=torch.int32, device=dev)
        self.W = (T + 63) // 64
        self.out = torch.empty_like(self.q)
        self.mask = torch.zeros((B, T, self.W), dtype=torch.int64, device=dev)
        self.ws_attn = _capi.tree_attention_workspace(self.q, self.kc, self.vc, self.mask, self.P,
                                                      self.nn)
        self.ws_ver = _capi.verify_workspace(B, T, dev)
        self.path = _capi.tree_attention_path(self.q, self.kc, self.vc, self.mask, self.P, self.nn)
        self.vout = (torch.zeros((B, T + 1), dtype=torch.int32, device=dev),
                     torch.zeros((B, T + 1), dtype=torch.int32, device=dev),
                     torch.zeros(B, dtype=torch.int32, device=dev))
        # own (default): the tree's K/V rows stay in their own [B][T][H][D]
        # tensors; K1 reads them there (st_attn_args.k_tree) and the commit
        # copies only the accepted rows into the cache — no K2 append of all T
        # rows. cache: K2 append into the cache scratch rows first, then
        # in-place compaction (the reference's cache discipline).
        self.own = tree_rows == "own"
        self.resident = (self.q, self.knew, self.vnew, self.tok, self.par, self.nn)

    def pre(self, a):
        qq, kn, vn, tk, pr, nd = a
        if self.own:   # ancestor masks; the previous kernel writes no input of theirs
            self.capi.build_masks(pr, nd, W=self.W, out=self.mask, early=True)
        else:          # K2 append + masks (one launch)
            self.capi.tree_prepare(kn, vn, self.P, nd, self.kc, self.vc, pr, W=self.W,
                                   out=self.mask)

    def k1(self, a):
        qq, kn, vn, tk, pr, nd = a
        # early_kv: the kernel right before K1 (masks / append+masks) writes
        # neither the prefix lengths nor committed rows [0, P), and the masks
        # kernel waits for ITS predecessor before it lets K1 start, so K1
        # streams the committed rows while the masks kernel runs
        self.capi.tree_attention(qq, self.kc, self.vc, self.mask, self.P, nd, out=self.out,
                                 workspace=self.ws_attn, k_tree=kn if self.own else None,
                                 v_tree=vn if self.own else None, early_kv=True)

    def post(self, a):   # K3 argmax, then the walk fused with the K2 commit
        qq, kn, vn, tk, pr, nd = a
        self.capi.verify_greedy_compact(self.logits, tk, pr, nd, self.P, self.kc, self.vc,
                                        workspace=self.ws_ver, want_argmax=False, out=self.vout,
                                        k_tree=kn if self.own else None,
                                        v_tree=vn if self.own else None)

    def run(self, a=None):
        a = a or self.resident
        self.pre(a)
        self.k1(a)
        self.post(a)

    def plan(self, a=None):
        """The same step as a native plan (st_verify_plan: the four launches
        issued by C++ with programmatic dependent launch; consecutive runs
        chain across steps, K1's tensor maps encoded once)."""
        qq, kn, vn, tk, pr, nd = a or self.resident
        return self.capi.VerifyPlan(qq, self.kc, self.vc, self.mask, self.P, nd, self.out,
                                    self.ws_attn, tk, pr, self.logits, self.ws_ver, *self.vout,
                                    k_tree=kn if self.own else None,
                                    v_tree=vn if self.own else None,
                                    k_new=None if self.own else kn,
                                    v_new=None if self.own else vn, early_kv=True)

    def k1_bytes(self, s=2):
        """Algorithmic K1 bytes per launch."""
        B_, T_, H_, D_, L_ = self.B, self.T, self.H, self.D, self.L
        return (s * (2 * B_ * L_ * H_ * D_ + B_ * T_ * H_ * D_ + 2 * B_ * T_ * H_ * D_
                     + B_ * T_ * H_ * D_) + 8 * B_ * T_ * self.W)

    def oracle_check(self):
        """Bench self-check (the oracle as CHECKER): the step's accepted
        tokens, node ids and lengths vs the CPU restatement's greedy verify
        (reference argmax_token + verify) on the same logits, bit-exact."""
        from oracle.oracle import Restatement
        R = Restatement()
        lg = self.logits.cpu().numpy()
        ver, ids, ln = (x.cpu().numpy() for x in self.vout)
        bad = 0
        for b in range(self.B):
            n = int(self.batch.n_nodes[b])
            _, rv, rids = R.greedy_verify(lg[b, :n], self.batch.tokens[b, :n],
                                          self.batch.parents[b, :n])
            if not (ln[b] == len(rv) and np.array_equal(ver[b, :ln[b]], rv)
                    and np.array_equal(ids[b, :ln[b]], rids)):
                bad += 1
        return {"greedy_vs_oracle": "bit-exact" if bad == 0 else f"MISMATCH in {bad} requests",
                "requests": self.B, "accepted_tokens": int(ln.sum())}


# ----------------------------------------------------------- reference arm ---
def reference_sample(n_threads, steps, warmup, full_tree, n_req=None):
    """The reference's own tree_parallel_decode (oracle/_ref, compiled from the
    unmodified reference sources) at the C2 layer shape on host cores.
    Reference recipe at LLaMA-7B attention shape: 1 layer, d=4096, 32 heads,
    V=258, ffn_mult=1; KV injected, one request per thread.
    full_tree: every request decodes its whole 64-node C2 tree; else a 9-node
    sample (root + one 8-deep path). Warm-up steps always use the 9-node
    sample (they only warm code and caches)."""
    from oracle.oracle import Reference, available_reference
    if not available_reference():
        return None
    R = Reference()

    class _T:
        def __init__(self, seqs):
            self.size = len(R.merge(seqs, 1 << 20)[0])

    n_req = n_req or n_threads
    trees = c2_trees(lambda s: _T(s), 7, 258, n_req=1)
    full = trees[0][1]
    sample = [full[0]]
    cfg = (1, H, H * D, 258, L + T + 2, 1)
    times = []
    for i in range(warmup + steps):
        seqs = full if (full_tree and i >= warmup) else sample
        t = R.bench_tree_decode(cfg, 42, n_req, L + 1, seqs, 1 << 20, n_threads)
        if i >= warmup:
            times.append(t)
    sec = statistics.median(times)
    seqs = full if full_tree else sample
    nodes = len(R.merge(seqs, 1 << 20)[0])
    return dict(value=n_req * nodes / sec, seconds=sec, nodes=nodes, requests=n_req,
                kind="reference", times=times)


def run_reference_arm(args):
    """The reference's CPU path on the SAME config as our arm (C2: 8 requests
    x 64-node trees over 2048 committed rows), all host threads (one request
    per thread — the reference decodes a request single-threaded)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    nt = cpu_threads()
    res = reference_sample(min(B, nt), args.steps, args.warmup, full_tree=True, n_req=B)
    cfg = {"workload": "C2 reference CPU path: tree_parallel_decode (f64) of 8 requests x "
                       "64-node trees over 2048 committed KV rows, LLaMA-7B attention-layer shape "
                       "(1 layer, d=4096, H=32; reference recipe V=258, ffn_mult=1)",
           "B": B, "T": T, "L": L, "H": H, "D": D, "same_config": True}
    if res is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (needs "
                          "/root/reference at build time)"}))
        return
    small = reference_sample(min(B, nt), 1, 0, full_tree=False, n_req=min(B, nt))
    sample = (f"{res['requests']} requests x full {res['nodes']}-node C2 tree (KV 2048) per step, "
              f"one request per host thread ({min(B, nt)} threads)")
    line = {"impl": "reference", "metric": METRIC, "value": res["value"], "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": res["seconds"] * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg,
            "cpu_baseline": {"value": res["value"], "unit": UNIT, "cores": min(B, nt),
                             "kind": "reference", "sample": sample},
            "e2e": {"value": res["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "sample_9node": {"value": small["value"], "ms_per_step": small["seconds"] * 1e3,
                             "note": "root + one 8-deep path per request (the round-1 arm)"}
            if small else None}
    print(json.dumps(line))


# -------------------------------------------------------------- clocks ----
class ClockSampler:
    def __init__(self, gpu_index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={gpu_index}", f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = []
        for line in open(self.f.name):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = max(float(r[2]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        loaded = [s for s in sm if s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows)}


def load_peaks():
    pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
    return json.load(open(pk)) if os.path.exists(pk) else {}


# ------------------------------------------------------- DP step runner ----
class DPRunner:
    """Replays a VerifyStep as CUDA graphs and, for N > 1, all-gathers every
    rank's accepted tokens + lengths (the DP exchange step)
    on a side stream: step i's exchange overlaps step i+1's compute (the next
    step of a rank needs only its own requests' results). The step's packed
    results are double-buffered so the exchange never races the next step."""

    def __init__(self, step, world, dev, native=True):
        import torch
        self.torch = torch
        self.native = native
        self.s, self.world = step, world
        Bs, Ts = step.B, step.T
        n = Bs * (Ts + 2)
        self.send = [torch.zeros(n, dtype=torch.int32, device=dev) for _ in range(2)]
        self.gathered = [torch.zeros(world * n, dtype=torch.int32, device=dev) for _ in range(2)]
        self.comm = torch.cuda.Stream() if world > 1 else None
        self.ev_ready = [torch.cuda.Event() for _ in range(2)]
        self.ev_sent = [torch.cuda.Event() for _ in range(2)]
        self.i = 0
        self.graphs = []
        self.ev_k1 = None

    def _pack(self, slot):
        ver, _, ln = self.s.vout
        Bs, Ts = self.s.B, self.s.T
        self.send[slot][: Bs * (Ts + 1)].copy_(ver.view(-1))
        self.send[slot][Bs * (Ts + 1):].copy_(ln)

    def capture(self, warmup, timed_k1=False):
        torch = self.torch
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(max(warmup, 3)):
                self.s.run()
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        if self.native:
            self.plan = self.s.plan()
            self.plan.run()
            torch.cuda.synchronize()
        for slot in range(2):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self.s.run()
                self._pack(slot)
            self.graphs.append(g)
        if timed_k1:  # the same step with timing events bracketing K1 (graph nodes)
            self.ev_k1 = (torch.cuda.Event(enable_timing=True, external=True),
                          torch.cuda.Event(enable_timing=True, external=True))
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                a = self.s.resident
                self.s.pre(a)
                self.ev_k1[0].record()
                self.s.k1(a)
                self.ev_k1[1].record()
                self.s.post(a)
            self.g_k1 = g

    def step(self, graph=None):
        """One step on the current stream (+ the exchange on the side stream)."""
        torch = self.torch
        slot = self.i % 2
        cur = torch.cuda.current_stream()
        if self.world > 1:
            cur.wait_event(self.ev_sent[slot])   # step i-2's exchange has read send[slot]
        if graph is None and self.native:
            self.plan.run()
            if self.world > 1:
                self._pack(slot)
        else:
            (graph or self.graphs[slot]).replay()
            if graph is not None:
                self._pack(slot)
        if self.world > 1:
            import torch.distributed as dist
            self.ev_ready[slot].record(cur)
            with torch.cuda.stream(self.comm):
                self.comm.wait_event(self.ev_ready[slot])
                dist.all_gather_into_tensor(self.gathered[slot], self.send[slot])
                self.ev_sent[slot].record(self.comm)
        self.i += 1

    def sync(self):
        torch = self.torch
        if self.comm is not None:
            torch.cuda.current_stream().wait_stream(self.comm)


def barrier_of(world):
    import torch
    import torch.distributed as dist

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
    return barrier


def max_over_ranks(world, dev, *vals):
    import torch
    import torch.distributed as dist
    if world == 1:
        return vals
    tt = torch.tensor(vals, dtype=torch.float64, device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    return tuple(tt.tolist())


def time_steps(runner, steps, barrier):
    import torch
    barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(steps):
        runner.step()
    runner.sync()
    t1.record()
    barrier()
    return t0.elapsed_time(t1)


def k1_alone_ms(step, steps, barrier):
    """K1's average launch duration: R back-to-back launches per graph replay,
    alternating between two KV/Q copies (each larger than L2, so no launch reads
    what the previous one left in L2); CUDA events around K replays on the
    launching stream."""
    import torch
    capi = step.capi
    kv2 = (step.kc.clone(), step.vc.clone(), step.q.clone())
    o2 = torch.empty_like(step.out)
    R_B2B = 8
    kt = step.knew if step.own else None
    vt = step.vnew if step.own else None

    def k1_b2b():
        for i in range(R_B2B):
            kk, vv, qq = (step.kc, step.vc, step.q) if i % 2 == 0 else kv2
            capi.tree_attention(qq, kk, vv, step.mask, step.P, step.nn,
                                out=step.out if i % 2 == 0 else o2, workspace=step.ws_attn,
                                k_tree=kt, v_tree=vt)
    k1_b2b()
    g_ = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_):
        k1_b2b()
    for _ in range(3):
        g_.replay()
    barrier()
    b0 = torch.cuda.Event(enable_timing=True)
    b1 = torch.cuda.Event(enable_timing=True)
    b0.record()
    for _ in range(steps):
        g_.replay()
    b1.record()
    barrier()
    ms = b0.elapsed_time(b1) / (steps * R_B2B)
    del kv2, o2, g_
    return ms


# ------------------------------------------------------------ our arm ------
def main():
    args = parse()
    if maybe_spawn(args):
        return
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.config == "c3":
        return run_c3(args)
    if args.config == "c4":
        return run_c4(args)
    if args.config == "c3e":
        return run_c3e(args)
    return run_verify(args)


def run_verify(args):
    """C2 (default) and C5: the verification step, requests partitioned over
    the ranks (weak scaling: B per GPU fixed)."""
    import torch

    rank, world, local, dev = init_rank(args)
    numa_cpus = bind_to_gpu_numa(local)
    c5 = args.config == "c5"
    Bq, Tq, Lq = (16, args.tree, args.kv) if c5 else (B, T, L)
    step = VerifyStep(dev, rank, B=Bq, T=Tq, L=Lq, tree_rows=args.tree_rows)
    barrier = barrier_of(world)
    runner = DPRunner(step, world, dev)
    runner.capture(args.warmup, timed_k1=True)
    for _ in range(max(args.warmup, 3)):
        runner.step()
    runner.sync()
    barrier()

    clocks = ClockSampler(local)
    # keep the GPU busy until the sampler reports (nvidia-smi needs ~0.2-0.5 s to start)
    soak_end = time.time() + 1.0
    while time.time() < soak_end:
        for _ in range(50):
            runner.step()
        runner.sync()
        torch.cuda.synchronize()
    ms = time_steps(runner, args.steps, barrier)
    runner.native = False   # the same step as one CUDA-graph replay per step (reported)
    ms_graph = time_steps(runner, args.steps, barrier)
    runner.native = True
    # K1 inside the step: the same K steps again from the graph whose timing
    # events bracket K1 on the launching stream
    k1_events = []
    for _ in range(args.steps):
        runner.step(graph=runner.g_k1)
        runner.ev_k1[1].synchronize()
        k1_events.append(runner.ev_k1[0].elapsed_time(runner.ev_k1[1]))
    runner.sync()
    k1_b2b_ms = k1_alone_ms(step, args.steps, barrier)
    for _ in range(200):        # keep sampling a little past the timed region
        runner.step()
    runner.sync()
    barrier()
    clk = clocks.stop()
    k1_ms = statistics.mean(k1_events)
    ms, k1_ms, k1_b2b_ms, ms_graph = max_over_ranks(world, dev, ms, k1_ms, k1_b2b_ms, ms_graph)
    ms_step = ms / args.steps
    value = Bq * Tq * world / (ms_step / 1e3)
    # this step's results vs the oracle (greedy verify, bit-exact) — rank 0 checks
    # its own requests after the timed region
    parity = step.oracle_check() if rank == 0 else None

    # ---- strong-scaling companion: STRONG_B_GLOBAL requests split over the ranks ----
    strong = None
    if not c5 and not args.no_strong and STRONG_B_GLOBAL % world == 0:
        del runner
        sb = STRONG_B_GLOBAL // world
        st2 = VerifyStep(dev, 100 + rank, B=sb, T=Tq, L=Lq, tree_rows=args.tree_rows)
        r2 = DPRunner(st2, world, dev)
        r2.capture(args.warmup)
        for _ in range(max(args.warmup, 3)):
            r2.step()
        r2.sync()
        (ms2,) = max_over_ranks(world, dev, time_steps(r2, args.steps, barrier))
        strong = {"B_global": STRONG_B_GLOBAL, "B_per_gpu": sb, "scaling": "strong",
                  "value": STRONG_B_GLOBAL * Tq / (ms2 / args.steps / 1e3), "unit": UNIT,
                  "ms_per_step": ms2 / args.steps}
        del r2, st2
        torch.cuda.empty_cache()
        runner = DPRunner(step, world, dev)
        runner.capture(0)

    # ---- e2e: C-ABI calls with HOST buffers, copies inside the timed region ----
    e2e = run_e2e(args, step, runner, world, dev, barrier, numa_cpus)

    # ---- roofline of the dominant kernel (K1) ----
    bytes_k1 = step.k1_bytes()
    achieved = bytes_k1 / (k1_b2b_ms / 1e3) / 1e9
    peak = load_peaks().get("hbm_gbs", 6553.6)
    traffic = None
    tf = os.path.join(ROOT, "profiles", "k1_traffic.json")
    if os.path.exists(tf) and not c5:
        traffic = json.load(open(tf)).get("dram_bytes_per_launch")

    if rank != 0:
        finish_rank(world)
        return

    cpu = None
    if world == 1 and not args.no_cpu_baseline and not c5:
        if _ORIG_AFFINITY:   # the CPU baseline gets every host core again
            os.sched_setaffinity(0, _ORIG_AFFINITY)
        nt = cpu_threads()
        try:
            res = reference_sample(min(B, nt), 1, 0, full_tree=True, n_req=B)
        except Exception as e:  # noqa: BLE001
            res = None
            print(f"cpu baseline failed: {e}", file=sys.stderr)
        if res is not None:
            cpu = {"value": res["value"], "unit": UNIT, "cores": min(B, nt), "kind": "reference",
                   "sample": f"{res['requests']} C2 requests (full {res['nodes']}-node tree, KV "
                             f"2048) through the reference tree_parallel_decode, f64, 1 layer "
                             f"d=4096 H=32 V=258 ffn_mult=1, one request per thread; "
                             f"{res['seconds']:.1f} s"}

    if c5:
        workload = (f"C5: LLaMA-7B-shape attention layer, fp16, batch 16/GPU, {Tq}-node tree, "
                    f"KV {Lq}, greedy verify (V=32000)")
    else:
        workload = ("C2: LLaMA-7B-shape attention layer, fp16, batch 8/GPU, 64-node tree, "
                    "KV 2048, greedy verify (V=32000)")
    kvmb = 2 * Bq * H * (Lq + Tq) * D * 2 / 1e6
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f16", "data": "synthetic",
        "config": {"workload": workload, "B_per_gpu": Bq, "T": Tq, "L": Lq, "H": H, "D": D, "V": V,
                   "parallelism": f"dp{world} (requests partitioned)",
                   "l2": f"inputs larger than L2: {kvmb:.0f} MB KV + {Bq * Tq * V * 4 / 1e6:.1f} MB "
                         f"logits per step",
                   "timing": "value: K steps, each one st_verify_plan_run (the step's four "
                             "launches issued natively with programmatic dependent launch, "
                             "chaining across steps; N>1: + the accepted-token all-gather on a "
                             "side stream, overlapping the next step), CUDA events around the K "
                             "steps; graph_ms_per_step: the same step as one CUDA-graph replay "
                             "per step; roofline: K replays of a graph of 8 back-to-back K1 "
                             "launches alternating between two KV/Q copies (> L2), CUDA events "
                             "around the replays; in-step bracket (event graph nodes around K1 "
                             "inside the step) reported beside it",
                   "k1_path": "tcgen05" if step.path == 2 else "cuda-core",
                   "tree_rows": args.tree_rows},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "K1 tree attention", "bytes_per_launch": bytes_k1,
                     "us_per_launch": k1_b2b_ms * 1e3,
                     "us_in_step_bracket": k1_ms * 1e3,
                     "share_of_step": k1_b2b_ms / ms_step,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)"},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": LAUNCHES_PER_STEP * args.steps,
        "clocks": clk,
        "parity": parity,
        "strong": strong,
        "graph_ms_per_step": ms_graph / args.steps,
        "verify_steps_per_s": 1e3 / ms_step,
        "node_evals_per_s": value,
        "verified_tokens_per_step": parity["accepted_tokens"] if parity else None,
    }
    if parity:
        line["verified_tokens_per_s"] = parity["accepted_tokens"] * world / (ms_step / 1e3)
    print(json.dumps(line), flush=True)
    finish_rank(world)
    if parity and parity["greedy_vs_oracle"] != "bit-exact":
        sys.exit(3)


def run_e2e(args, step, runner, world, dev, barrier, numa_cpus):
    """Per step: the host merges every request's candidate sequences into its
    tree (st_tree_merge_batch, thread pool, packed into pinned memory), H2D of
    Q, the tree's K/V and the topology, the step, D2H of the accepted tokens +
    lengths, which the host reads. Serving-style pipelining: step i+1's merge +
    H2D run while step i computes (two host and two device input sets)."""
    import torch

    from paper_2305_09781_b200.tree import MergeInputs, merge_batch
    Bq, Tq = step.B, step.T
    merge_in = MergeInputs([sq for _, sq in step.trees])
    h_q = step.q.cpu().pin_memory()
    h_k = step.knew.cpu().pin_memory()
    h_v = step.vnew.cpu().pin_memory()
    h_topos = [torch.empty(2 * Bq * Tq + Bq, dtype=torch.int32).pin_memory() for _ in range(2)]

    def host_merge(h):
        merge_batch(merge_in, Tq, max_nodes=Tq,
                    out=(h[: Bq * Tq].view(Bq, Tq), h[Bq * Tq: 2 * Bq * Tq].view(Bq, Tq), None,
                         h[2 * Bq * Tq:]))
    for h in h_topos:
        host_merge(h)
        assert np.array_equal(h[: Bq * Tq].numpy().reshape(Bq, Tq), step.batch.tokens)
        assert np.array_equal(h[2 * Bq * Tq:].numpy(), step.batch.n_nodes)
    t_m = time.perf_counter()
    for _ in range(50):
        host_merge(h_topos[1])
    merge_us = (time.perf_counter() - t_m) / 50 * 1e6
    h_topo = h_topos[0]
    h2d = (h_q.numel() * 2 + h_k.numel() * 2 + h_v.numel() * 2 + h_topo.numel() * 4)
    sets = []
    for _ in range(2):
        topo = torch.empty_like(h_topo, device=dev)
        sets.append((torch.empty_like(step.q), torch.empty_like(step.knew),
                     torch.empty_like(step.vnew), topo[: Bq * Tq].view(Bq, Tq),
                     topo[Bq * Tq: 2 * Bq * Tq].view(Bq, Tq), topo[2 * Bq * Tq:], topo))
    h_outs = [torch.empty(Bq * (Tq + 1) + Bq, dtype=torch.int32).pin_memory() for _ in range(2)]
    d2h = h_outs[0].numel() * 4
    # the H2D of a step is split over two copy streams (two copy engines): a
    # single stream leaves PCIe headroom on some hosts (ST_E2E_STREAMS=1: one)
    n_cs = max(1, int(os.environ.get("ST_E2E_STREAMS", "2")))
    copy_streams = [torch.cuda.Stream() for _ in range(n_cs)]
    copy_stream = copy_streams[0]
    ev_copied_cs = [[torch.cuda.Event() for _ in range(n_cs)] for _ in range(2)]
    ev_copied = [torch.cuda.Event() for _ in range(2)]
    ev_free = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]
    for st in sets:   # warm + capture one full-step graph per input set
        st[6].copy_(h_topo)
        st[0].copy_(h_q), st[1].copy_(h_k), st[2].copy_(h_v)
    plans = [step.plan(st[:6]) for st in sets]   # one prepared step per input set
    cur = torch.cuda.current_stream()

    def issue_copy(i, merge=True):
        st = sets[i % 2]
        h = h_topos[i % 2]
        if merge:   # host buffer i%2 was last read by step i-2's copy
            ev_copied[i % 2].synchronize()
            host_merge(h)
        # each of Q, K, V split into n_cs row ranges, one per copy stream
        for j, cs in enumerate(copy_streams):
            with torch.cuda.stream(cs):
                cs.wait_event(ev_free[i % 2])
                for dst, src in ((st[0], h_q), (st[1], h_k), (st[2], h_v)):
                    d_, s_ = dst.view(-1), src.view(-1)
                    n_ = d_.numel()
                    a_, b_ = n_ * j // n_cs, n_ * (j + 1) // n_cs
                    d_[a_:b_].copy_(s_[a_:b_], non_blocking=True)
                if j == 0:
                    st[6].copy_(h, non_blocking=True)
                ev_copied_cs[i % 2][j].record(cs)
        with torch.cuda.stream(copy_stream):
            for j in range(1, n_cs):
                copy_stream.wait_event(ev_copied_cs[i % 2][j])
            ev_copied[i % 2].record(copy_stream)

    def issue_compute(i):
        cur.wait_event(ev_copied[i % 2])
        plans[i % 2].run()
        ev_free[i % 2].record(cur)
        if world > 1:   # DP exchange, synchronous here: the host reads the gathered result
            import torch.distributed as dist
            runner._pack(0)
            dist.all_gather_into_tensor(runner.gathered[0], runner.send[0])
            h_outs[i % 2].copy_(runner.gathered[0][: h_outs[0].numel()], non_blocking=True)
        else:
            h_outs[i % 2][: Bq * (Tq + 1)].copy_(step.vout[0].view(-1), non_blocking=True)
            h_outs[i % 2][Bq * (Tq + 1):].copy_(step.vout[2], non_blocking=True)
        ev_out[i % 2].record(cur)

    def read_result(i):
        ev_out[i % 2].synchronize()
        return int(h_outs[i % 2][Bq * (Tq + 1):].sum())   # host consumes the accepted lengths

    def e2e_run(n):
        got = 0
        issue_copy(0)
        for i in range(n):
            if i + 1 < n:
                issue_copy(i + 1)
            issue_compute(i)
            if i >= 1:
                got += read_result(i - 1)
        got += read_result(n - 1)
        return got

    e2e_run(4)
    # the copies alone, event-timed on the copy stream: explains e2e (PCIe-bound)
    barrier()
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record(copy_stream)
    for i in range(10):
        issue_copy(i, merge=False)
    c1.record(copy_stream)
    barrier()
    h2d_gbs = h2d * 10 / (c0.elapsed_time(c1) / 1e3) / 1e9
    # three windows of K end-to-end steps; the median window is reported
    windows = []
    for _ in range(3):
        barrier()
        w0 = time.perf_counter()
        e2e_run(args.steps)
        barrier()
        windows.append((time.perf_counter() - w0) * 1e3)
    (e2e_ms,) = max_over_ranks(world, dev, statistics.median(windows))
    return {"value": Bq * Tq * world / (e2e_ms / args.steps / 1e3), "unit": UNIT,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ms_per_step": e2e_ms / args.steps,
            "windows_ms_per_step": [w / args.steps for w in windows],
            "h2d_gbs_copies_alone": h2d_gbs,
            "h2d_copy_streams": n_cs,
            "h2d_gbs_implied": h2d / (e2e_ms / args.steps / 1e3) / 1e9,
            "host_numa_cpus": numa_cpus,
            "host_tree_merge_us_per_step": merge_us,
            "note": "per step: host merge_sequences of all B trees on the thread pool into "
                    "pinned memory + H2D, pipelined against the previous step's compute; "
                    "bound by PCIe H2D"}


# ------------------------------------------------------------------ C4 -----
def run_c4(args):
    """C4 (BASELINE.json configs[3]): LLaMA-65B-shape attention layer (64 heads x
    128, fp16), 8 requests with merged trees of 3 SSMs expanded
    <1,1,3,1,1,1,1,1> (61 nodes), KV 2048, heads sharded over the ranks
    (64/N per rank). One step = masks -> K1 over this rank's heads -> the
    head-output all-gather to [B][T][64][128] on every rank (NCCL
    all_gather_into_tensor + layout kernel, or --gather peer: fused into K1's
    epilogue over peer memory) -> greedy verify (V=32000, replicated). Strong
    scaling: the layer's work is fixed, N splits its heads."""
    import torch

    from paper_2305_09781_b200 import _capi
    from paper_2305_09781_b200.dist import PeerHeadGather, gather_head_outputs, head_shard
    from paper_2305_09781_b200.tree import TokenTree, TreeBatch

    rank, world, local, dev = init_rank(args)
    HT, Bq = 64, 8
    h0, h1 = head_shard(HT, world, rank)
    Hl = h1 - h0
    trees = c4_trees(lambda s: TokenTree.merge_sequences(s, 1 << 20), 65, Bq)
    tb = TreeBatch([t for t, _ in trees])
    Tq = tb.T
    g = torch.Generator(device=dev).manual_seed(99 + rank)
    q = (torch.rand(Bq, Tq, Hl, D, device=dev, generator=g) * 2 - 1).half()
    kc = (torch.rand(Bq, Hl, L + Tq, D, device=dev, generator=g) * 2 - 1).half()
    vc = (torch.rand(Bq, Hl, L + Tq, D, device=dev, generator=g) * 2 - 1).half()
    kt = (torch.rand(Bq, Tq, Hl, D, device=dev, generator=g) * 2 - 1).half()
    vt = (torch.rand(Bq, Tq, Hl, D, device=dev, generator=g) * 2 - 1).half()
    g2 = torch.Generator(device=dev).manual_seed(5)   # same logits on every rank
    logits = torch.randn(Bq, Tq, V, device=dev, generator=g2)
    par = torch.tensor(tb.parents, device=dev)
    tok = torch.tensor(tb.tokens, device=dev)
    nn = torch.tensor(tb.n_nodes, device=dev)
    P = torch.full((Bq,), L, dtype=torch.int32, device=dev)
    mask = _capi.build_masks(par, nn)
    out = torch.empty_like(q)
    ws = _capi.tree_attention_workspace(q, kc, vc, mask, P, nn)
    wsv = _capi.verify_workspace(Bq, Tq, dev)
    gathered = torch.empty((world, Bq, Tq, Hl, D), dtype=torch.float16, device=dev)
    full = torch.empty((Bq, Tq, HT, D), dtype=torch.float16, device=dev)
    vout = (torch.zeros((Bq, Tq + 1), dtype=torch.int32, device=dev),
            torch.zeros((Bq, Tq + 1), dtype=torch.int32, device=dev),
            torch.zeros(Bq, dtype=torch.int32, device=dev))
    peer = None
    if args.gather == "peer" and world > 1:
        peer = PeerHeadGather(Bq, Tq, Hl, D, torch.float16, dev, world, rank)
    barrier = barrier_of(world)

    def step():
        _capi.build_masks(par, nn, out=mask)
        if peer is not None:
            peer.attention(q, kc, vc, mask, P, nn, workspace=ws)
            o = peer.wait()
        else:
            _capi.tree_attention(q, kc, vc, mask, P, nn, out=out, workspace=ws, k_tree=kt,
                                 v_tree=vt)
            o = gather_head_outputs(out, world, gathered=gathered, out=full)
        _capi.verify_greedy(logits, tok, par, nn, workspace=wsv, want_argmax=False, out=vout)
        return o

    for _ in range(max(args.warmup, 3)):
        step()
    barrier()
    clocks = ClockSampler(local)
    time.sleep(0.5)
    barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(args.steps):
        step()
    t1.record()
    barrier()
    clk = clocks.stop()
    (ms,) = max_over_ranks(world, dev, t0.elapsed_time(t1))
    ms_step = ms / args.steps
    bytes_k1 = 2 * (2 * Bq * L * Hl * D + Bq * Tq * Hl * D + 2 * Bq * Tq * Hl * D
                    + Bq * Tq * Hl * D) + 8 * Bq * Tq
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": Bq * Tq / (ms_step / 1e3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f16",
            "data": "synthetic",
            "config": {"workload": "C4: LLaMA-65B-shape attention layer (64 heads), heads sharded "
                                   "over the GPUs, B=8, merged 3-SSM trees <1,1,3,1,1,1,1,1>, KV "
                                   "2048, head-output all-gather + greedy verify",
                       "B": Bq, "T": Tq, "L": L, "H_total": HT, "H_per_gpu": Hl,
                       "gather": args.gather if world > 1 else "none (1 rank)",
                       "parallelism": f"heads/{world}"},
            "k1_bytes_per_gpu": bytes_k1,
            "gather_bytes_received_per_gpu": (world - 1) * Bq * Tq * Hl * D * 2,
            "gpu_launches": args.steps * (4 if peer is None else 4),
            "clocks": clk}))
    finish_rank(world)


# ------------------------------------------------------------------ C3 -----
def run_c3(args):
    """C3 (BASELINE.json configs[2]): LLaMA-7B-shape full decoder stack (reference
    recipe: 32 layers, d=4096, 32 heads, FFN x4, V=32000, learned positions), a
    global batch of 32 requests partitioned over the ranks (strong scaling),
    64-node trees over 2048 committed rows, stochastic multi-step speculative
    sampling (K4). One step = tree embedding -> 32 x [LN, QKV GEMM (tree K/V
    kept per layer), K1 (k_tree mode), WO/FFN GEMMs with fused GELU / residual]
    -> LM head -> K4 MSS verify -> K2 commit of the accepted rows of all 32
    layers (+ accepted-token all-gather for N > 1). Synthetic KV prefix and draft
    distributions; weights generated on the GPU from UniformStream(42)."""
    import torch

    from paper_2305_09781_b200 import _capi
    from paper_2305_09781_b200.dist import gather_accepted, shard_range
    from paper_2305_09781_b200.tree import TokenTree, TreeBatch

    rank, world, local, dev = init_rank(args)
    NL, d, Hh, Vv, BG = 32, 4096, 32, 32000, 32
    lo, hi = shard_range(BG, world, rank)
    Bl = hi - lo
    model = _capi.DeviceModel(NL, Hh, d, Vv, L + T + 64, 4, seed=42, dtype=torch.float16)
    Lmax = L + T
    kc, vc = model.new_cache(Bl, Lmax)
    kc.uniform_(-1, 1)
    vc.uniform_(-1, 1)
    trees = c2_trees(lambda s_: TokenTree.merge_sequences(s_, 1 << 20), 3000 + lo, Vv, n_req=Bl)
    batch = TreeBatch([t for t, _ in trees], T)
    tok = torch.tensor(batch.tokens, device=dev)
    par = torch.tensor(batch.parents, device=dev)
    nn = torch.tensor(batch.n_nodes, device=dev)
    P = torch.full((Bl,), L, dtype=torch.int32, device=dev)
    pos = (P[:, None] + torch.tensor(batch.depths, device=dev)).to(torch.int32)
    mask = _capi.build_masks(par, nn)
    g = torch.Generator(device=dev).manual_seed(7 + rank)
    qd = torch.softmax(torch.randn(Bl, T, Vv, device=dev, generator=g) * 3, dim=-1)
    U = torch.rand(Bl, T + 1, device=dev, generator=g)
    logits = torch.empty(Bl, T, Vv, dtype=torch.float32, device=dev)
    gathered = torch.zeros(world * Bl * (T + 2), dtype=torch.int32, device=dev)

    # k_tree mode: every layer's tree K/V stay in tree_qkv (no per-layer
    # append); the accepted rows of all 32 layers are committed from there
    tree_qkv = model.new_tree_qkv(Bl, T)

    def step():
        model.tree_forward(tok, pos, mask, P, nn, kc, vc, logits=logits, tree_qkv=tree_qkv)
        ver, ids, ln = _capi.verify_mss(logits, qd, tok, par, nn, 1.0, U)
        _capi.kv_commit_tree(ids, ln, P, tree_qkv, kc, vc, T)
        if world > 1:
            gather_accepted(ver, ln, world, out=gathered)
        return ln

    barrier = barrier_of(world)
    for _ in range(max(args.warmup, 2)):
        ln = step()
    barrier()
    clocks = ClockSampler(local)
    time.sleep(0.5)
    barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(args.steps):
        ln = step()
    t1.record()
    barrier()
    clk = clocks.stop()
    (ms,) = max_over_ranks(world, dev, t0.elapsed_time(t1))
    ms_step = ms / args.steps
    accepted = int(ln.sum().item())
    wbytes = model.param_count * 2
    kvbytes = NL * 2 * Bl * Hh * L * (d // Hh) * 2
    # algorithmic FLOPs per step per GPU: every projection over the B*T tree rows
    # (QKV+WO 4d^2, FFN 2*4d^2 per layer; LM head d*V) + attention QK^T and PV
    # over the L+T visible-or-masked rows (the dense MMA work K1 issues)
    rows = Bl * T
    gemm_flops = 2 * rows * (NL * 12 * d * d + d * Vv)
    attn_flops = NL * 4 * rows * d * (L + T)
    flops = gemm_flops + attn_flops
    tpeak = load_peaks().get("bf16_tflops_sustained", 1392.6)
    tach = flops / (ms_step / 1e3) / 1e12
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": BG * T / (ms_step / 1e3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f16",
            "data": "synthetic",
            "config": {"workload": "C3: LLaMA-7B-shape full decoder stack (reference recipe), batch "
                                   "32 partitioned over GPUs, 64-node trees, KV 2048, stochastic MSS",
                       "B_global": BG, "B_per_gpu": Bl, "T": T, "L": L, "layers": NL, "d": d,
                       "V": Vv, "parallelism": f"dp{world} (requests partitioned)"},
            "roofline": {"bound": "tensor", "achieved": tach, "peak": tpeak, "unit": "TFLOP/s",
                         "frac": tach / tpeak, "traffic": None,
                         "flops_per_step_per_gpu": flops, "gemm_flops": gemm_flops,
                         "attn_flops": attn_flops,
                         "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained (cuBLAS bf16; "
                                        "the step computes f16, same tensor-core rate)",
                         "hbm_bytes_per_step_per_gpu": wbytes + kvbytes,
                         "note": "whole-step figure: the GEMMs dominate (intensity ~ B*T rows)"},
            "verified_tokens_per_step": accepted * world, "clocks": clk}))
    finish_rank(world)


# ---------------------------------------------------------------- C3 e2e ----
def run_c3e(args):
    """C3 model shapes END TO END through the device-resident engine
    (st_engine): LLM = LLaMA-7B-shape stack (reference recipe: 32 layers,
    d=4096, 32 heads, FFN x4, V=32000), draft model = a 2-layer model of the
    same width, 32 requests partitioned over the ranks, 128-token prompts,
    expansion trees <1,1,3,1,1,1,1,1> drafted on the GPU, greedy tree
    verification, 64 new tokens per request. Timed: prompt upload + prefill +
    every step until all budgets are spent, with the per-step D2H read of the
    accepted tokens (what a serving loop does). Random weights: the draft model
    does not predict the LLM, so most steps accept the bonus token only — the
    number measures the engine's machinery at C3 shapes, not acceptance."""
    import torch

    from paper_2305_09781_b200 import _capi

    rank, world, local, dev = init_rank(args)
    NL, d, Hh, Vv, BG, PROMPT, NEW = 32, 4096, 32, 32000, 32, 128, 64
    lo = BG * rank // world
    Bl = BG * (rank + 1) // world - lo
    expansion = (1, 1, 3, 1, 1, 1, 1, 1)
    llm = _capi.DeviceModel(NL, Hh, d, Vv, PROMPT + NEW + 64, 4, seed=42, dtype=torch.float16)
    ssm = _capi.DeviceModel(2, Hh, d, Vv, PROMPT + NEW + 64, 4, seed=7, dtype=torch.float16)
    eng = _capi.Engine(llm, ssm, Bl, PROMPT, expansion=expansion)
    rng = np.random.default_rng(11 + rank)
    prompts = [rng.integers(0, Vv, PROMPT).tolist() for _ in range(Bl)]
    budgets = [NEW] * Bl
    barrier = barrier_of(world)
    eng.run(prompts, [4] * Bl)          # warm-up (kernel attributes, tensor maps)
    barrier()
    clocks = ClockSampler(local)
    time.sleep(0.5)
    barrier()
    t0 = time.perf_counter()
    seqs, steps = eng.run(prompts, budgets)
    barrier()
    wall = time.perf_counter() - t0
    clk = clocks.stop()
    generated = sum(len(q) - PROMPT for q in seqs)
    (wall, steps_max) = max_over_ranks(world, dev, wall, float(steps))
    total = generated * world if world > 1 else generated
    if rank == 0:
        print(json.dumps({
            "metric": "generated tokens/s (C3 shapes, device engine, end to end)",
            "value": total / wall, "unit": "tokens/s", "n_gpus": world, "steps": int(steps_max),
            "warmup": 1, "ms_per_step": wall / steps_max * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f16", "data": "synthetic",
            "config": {"workload": "C3 shapes through st_engine: 32-layer d=4096 LLM, 2-layer "
                                   "draft model, expansion <1,1,3,1,1,1,1,1> drafted on the GPU, "
                                   "greedy verification, 128-token prompts, 64 new tokens",
                       "B_global": BG, "B_per_gpu": Bl, "tree_nodes": eng.T,
                       "parallelism": f"dp{world} (requests partitioned)"},
            "tokens_per_step_per_request": generated / max(1, Bl) / max(1, steps),
            "e2e": {"value": total / wall, "unit": "tokens/s",
                    "h2d_bytes_per_step": 0, "d2h_bytes_per_step": (eng.T + 3) * Bl * 4,
                    "note": "prompts uploaded once; per step only the accepted tokens, lengths "
                            "and done flags come back"},
            "clocks": clk}))
    finish_rank(world)


if __name__ == "__main__":
    main()
