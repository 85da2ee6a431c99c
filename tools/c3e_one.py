"""One C3-shape device-engine run (prefill + 2 steps) for an ncu launch list:
  ncu --metrics gpu__time_duration.sum --csv python tools/c3e_one.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_09781_b200 import _capi  # noqa: E402

NL, d, Hh, Vv, B, PROMPT = 32, 4096, 32, 32000, 32, 128
llm = _capi.DeviceModel(NL, Hh, d, Vv, PROMPT + 64 + 64, 4, seed=42, dtype=torch.float16)
ssm = _capi.DeviceModel(2, Hh, d, Vv, PROMPT + 64 + 64, 4, seed=7, dtype=torch.float16)
eng = _capi.Engine(llm, ssm, B, PROMPT, expansion=(1, 1, 3, 1, 1, 1, 1, 1))
rng = np.random.default_rng(11)
prompts = [rng.integers(0, Vv, PROMPT).tolist() for _ in range(B)]
torch.cuda.synchronize()
seqs, steps = eng.run(prompts, [3] * B)
torch.cuda.synchronize()
print("steps", steps)
