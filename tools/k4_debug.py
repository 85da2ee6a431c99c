import numpy as np, torch, sys, os
sys.path.insert(0, os.getcwd())
from oracle.oracle import Restatement
from paper_2305_09781_b200 import _capi
from tests.test_mss import make_case
R = Restatement()
for V, tau in [(32000, 0.7), (32000, 1.0), (1000, 0.7), (4096, 0.7), (8192, 0.7), (16000, 0.7)]:
    rng = np.random.default_rng(V)
    tok, par, n, logits, q = make_case(R, rng, V, width=4, depth=5, n_req=6)
    Bq, T = tok.shape
    U = rng.uniform(0, 1, (Bq, T + 1)).astype(np.float32)
    dev = "cuda"
    ver, ids, ln = _capi.verify_mss(torch.tensor(logits, device=dev), torch.tensor(q, device=dev),
                                    torch.tensor(tok, device=dev), torch.tensor(par, device=dev),
                                    torch.tensor(n, device=dev), tau, torch.tensor(U, device=dev))
    ver, ids, ln = ver.cpu().numpy(), ids.cpu().numpy(), ln.cpu().numpy()
    bad = 0
    for b in range(Bq):
        k = n[b]
        rv, rids = R.mss_verify(logits[b, :k], q[b, :k], tok[b, :k], par[b, :k], tau, U[b])
        if ln[b] != len(rv) or list(ver[b, :ln[b]]) != list(rv) or list(ids[b, :ln[b]]) != list(rids):
            bad += 1
            print(V, tau, "req", b, "gpu", list(ids[b, :ln[b]]), list(ver[b, :ln[b]]), "ref", list(rids), list(rv))
    print(V, tau, "bad", bad, "of", Bq)
