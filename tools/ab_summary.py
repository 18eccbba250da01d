#!/usr/bin/env python
"""Median ms per launch (first launch dropped) per variant x case x dtype from tools/gpu_ab.sh output."""
import collections
import re
import statistics
import sys

rows = collections.defaultdict(list)
for line in open(sys.argv[1]):
    m = re.match(r"(\S+) (\S+) (\S+) (f32|f64) n=\d+ ms/launch=\[(.*)\]", line)
    if m:
        v, case, _, dt, arr = m.groups()
        t = [float(x.strip(" '")) for x in arr.split(",")][1:]
        rows[(case, dt, v)].extend(t)
for (case, dt, v), t in sorted(rows.items()):
    print(f"{case:4s} {dt} {v:10s} median {statistics.median(t):.4f} ms  (n={len(t)})")
