"""Device-resident f16 engine (st_engine_*: drafting on the GPU, LLM tree
verification, greedy walk + budget/EOS + commit on the device).

Exactness model: greedy speculative decoding must reproduce greedy
incremental decoding token for token (reference engine.cpp; acceptance
criterion #1). In f16 the same token path can get slightly different logits
in a tree pass than in an incremental pass (different GEMM row counts,
different attention tiling), so two runs may legitimately part ways where the
LLM's top-2 logit gap is within f16 noise. The tests compare sequences up to
the first generated position whose top-2 gap (from one f16 pass over the
incremental sequence) is below MARGIN, and require that prefix to cover most
of the run.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
MARGIN = 0.01   # f16 logit noise at these shapes is ~1e-3


@pytest.fixture(scope="module")
def capi():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2305_09781_b200 import _capi
    return _capi


def _model(capi, layers, heads, d, V, maxpos, seed):
    return capi.DeviceModel(layers, heads, d, V, maxpos, 4, seed=seed, dtype=torch.float16)


def _gaps(capi, model, seq):
    """top-2 logit gap at every position of seq (one causal f16 pass)."""
    dev = "cuda"
    n = len(seq)
    tok = torch.tensor([seq], dtype=torch.int32, device=dev)
    pos = torch.arange(n, dtype=torch.int32, device=dev)[None]
    par = (torch.arange(n, dtype=torch.int32, device=dev) - 1)[None]
    nn = torch.tensor([n], dtype=torch.int32, device=dev)
    mask = capi.build_masks(par, nn)
    kc, vc = model.new_cache(1, n + 8)
    P = torch.zeros(1, dtype=torch.int32, device=dev)
    lg = model.tree_forward(tok, pos, mask, P, nn, kc, vc)[0]
    top2 = torch.topk(lg, 2, dim=-1).values
    return (top2[:, 0] - top2[:, 1]).cpu().numpy()


def _agree(capi, model, a, b, prompt_len):
    """a, b agree up to the first low-margin generated position of a."""
    g = _gaps(capi, model, a)
    stop = len(a)
    for i in range(prompt_len - 1, len(a) - 1):   # logits at i predict token i+1
        if g[i] < MARGIN:
            stop = i + 1
            break
    n = min(stop, len(b))
    assert a[:n] == b[:n], f"diverged before the first low-margin position {stop}"
    return stop


PROMPTS = [[5, 9, 2, 7, 4], [1, 2, 3], [100, 200, 7, 7, 9, 11, 300], [42]]
BUDGETS = [40, 33, 29, 45]


def _cfg():
    return dict(layers=2, heads=4, d=512, V=512, maxpos=128)


def test_engine_incremental_and_self_speculation(capi):
    c = _cfg()
    llm = _model(capi, c["layers"], c["heads"], c["d"], c["V"], c["maxpos"], 31)
    inc = capi.Engine(llm, None, len(PROMPTS), 8, expansion=())
    seqs_inc, steps_inc = inc.run(PROMPTS, BUDGETS)
    assert steps_inc == max(BUDGETS)
    for p, b, s in zip(PROMPTS, BUDGETS, seqs_inc):
        assert len(s) == len(p) + b and s[: len(p)] == p
    spec = capi.Engine(llm, None, len(PROMPTS), 8, expansion=(1, 1, 1, 1))
    seqs_spec, steps_spec = spec.run(PROMPTS, BUDGETS)
    covered = 0
    for p, a, b in zip(PROMPTS, seqs_inc, seqs_spec):
        covered += _agree(capi, llm, a, b, len(p)) - len(p)
    assert covered >= 0.5 * sum(BUDGETS)
    # the LLM drafting for itself accepts the whole chain: 5 tokens per step
    assert steps_spec <= -(-max(BUDGETS) // 5) + 2


def test_engine_draft_model_trees_budget_eos(capi):
    c = _cfg()
    llm = _model(capi, c["layers"], c["heads"], c["d"], c["V"], c["maxpos"], 31)
    ssm = _model(capi, 1, c["heads"], c["d"], c["V"], c["maxpos"], 77)
    inc = capi.Engine(llm, None, len(PROMPTS), 8, expansion=())
    seqs_inc, _ = inc.run(PROMPTS, BUDGETS)
    eng = capi.Engine(llm, ssm, len(PROMPTS), 8, expansion=(2, 2, 1))
    assert eng.T == 1 + 2 + 4 + 4
    seqs, steps = eng.run(PROMPTS, BUDGETS)
    for p, a, b, bud in zip(PROMPTS, seqs_inc, seqs, BUDGETS):
        assert len(b) == len(p) + bud
        _agree(capi, llm, a, b, len(p))
    # EOS: cut right after the first occurrence of a token the run emits
    eos = seqs_inc[0][len(PROMPTS[0]) + 6]
    eng2 = capi.Engine(llm, ssm, len(PROMPTS), 8, expansion=(2, 2, 1), eos=eos)
    seqs_e, _ = eng2.run(PROMPTS, BUDGETS)
    for p, a, b, bud in zip(PROMPTS, seqs_inc, seqs_e, BUDGETS):
        gen = a[len(p):]
        want = a[: len(p) + (gen.index(eos) + 1 if eos in gen else bud)]
        stop = _agree(capi, llm, a, b, len(p))
        if stop >= len(want):
            assert b == want


@pytest.mark.parametrize("expansion", [(), (1, 1, 1, 1), (2, 2)])
def test_engine_matches_reference_engine_golden(capi, golden, expansion):
    """The f16 engine against the reference's own f64 run_incremental /
    run_speculative sequence (tests/golden/engine_c1.npz, C1 model shape, 24
    tokens), compared up to the first position whose REFERENCE f64 top-2 logit
    gap is below 5e-3 (fixture chosen so that all 24 are comparable)."""
    g = golden("engine_c1.npz")
    layers, heads, d, V, maxpos, ffn = (int(x) for x in g["cfg"])
    llm = capi.DeviceModel(layers, heads, d, V, maxpos, ffn, seed=int(g["seed"]),
                           dtype=torch.float16)
    prompt = g["prompt"].tolist()
    ref = g["incremental"].tolist()
    assert ref == g["speculative"].tolist()
    gaps = g["gaps"]
    stop = len(prompt) + (int(np.argmax(gaps < 5e-3)) if (gaps < 5e-3).any() else len(gaps))
    assert stop == len(ref)
    eng = capi.Engine(llm, None, 1, len(prompt), expansion=expansion)
    seqs, steps = eng.run([prompt], [len(ref) - len(prompt)])
    assert seqs[0][:stop] == ref[:stop]
    if expansion == (1, 1, 1, 1):   # same step count as the reference's perfect speculator
        assert steps == int(g["speculative_steps"])


def test_comm_single_rank_gather_accepted(capi):
    """st_comm_*: the C-ABI NCCL module (DP exchange). One GPU per call here
    (NCCL refuses two ranks on one device), so this checks the single-rank
    communicator end to end: unique id -> init -> gather_accepted packs the
    verified tokens + lengths exactly as the multi-rank layout expects."""
    uid = capi.Comm.unique_id()
    comm = capi.Comm(1, 0, uid)
    B, T = 5, 7
    ver = torch.randint(0, 1000, (B, T + 1), dtype=torch.int32, device="cuda")
    ln = torch.randint(1, T + 2, (B,), dtype=torch.int32, device="cuda")
    pack = torch.empty(B * (T + 2), dtype=torch.int32, device="cuda")
    gathered = torch.empty(1 * B * (T + 2), dtype=torch.int32, device="cuda")
    comm.gather_accepted(ver, ln, pack, gathered)
    torch.cuda.synchronize()
    assert torch.equal(gathered[: B * (T + 1)].view(B, T + 1), ver)
    assert torch.equal(gathered[B * (T + 1):], ln)


def test_engine_bf16_incremental_matches_speculative(capi):
    c = _cfg()
    llm = capi.DeviceModel(c["layers"], c["heads"], c["d"], c["V"], c["maxpos"], 4, seed=31,
                           dtype=torch.bfloat16)
    inc = capi.Engine(llm, None, len(PROMPTS), 8, expansion=())
    seqs_inc, _ = inc.run(PROMPTS, BUDGETS)
    spec = capi.Engine(llm, None, len(PROMPTS), 8, expansion=(2, 1, 1))
    seqs_spec, _ = spec.run(PROMPTS, BUDGETS)
    for p, a, b in zip(PROMPTS, seqs_inc, seqs_spec):
        assert len(b) == len(a)
        _agree(capi, llm, a, b, len(p))
