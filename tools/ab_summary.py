"""Summarise tools/gpu_ab_lib.sh output: per shape, each variant's times."""
import collections
import sys

d = collections.defaultdict(list)
order = []
for line in sys.stdin:
    if " us " not in line or "]" not in line:
        continue
    v = line.split()[0]
    head = line[:line.index(" us")]
    us = float(head.split()[-1])
    name = head[len(v):].split("]", 1)[1].rsplit(None, 1)[0].strip()
    d[(name, v)].append(us)
    if v not in order:
        order.append(v)
for n in sorted(set(k[0] for k in d)):
    print(f"{n:30s}", "  ".join(f"{v}: " + " ".join(f"{x:7.2f}" for x in d[(n, v)]) for v in order))
