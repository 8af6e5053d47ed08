#!/usr/bin/env python
"""SURVEY §8c pin P8 (no skipped or duplicated work): the DFMA thread-instructions ncu counts in one
launch of the split ring kernel (smsp__sass_thread_inst_executed_op_dfma_pred_on.sum, from
tools/gpurun_r2_evidence.sh) against the count the pattern predicts. For X^2 (alpha = 1, beta = 0:
the emission executes no DFMA) a step issues 64 G thread-DFMAs (G = 64-entry groups of the launch;
the accumulator loads and stores of a group past the B row's end are predicated off, its DFMAs are
not), and row i runs its nnz(i) steps in pieces of 64 - 2 HB + 1, each padded with null steps to whole
halves of HB steps. So DFMA = 64 G sum_i sum_pieces HB ceil(cnt / HB): every step of every row
executed exactly once. The products P = sum over steps of nnz(k) are reported beside it.

python tools/p8_dfma.py gpurun_out/dfma.csv N M [G HB]   (G, HB of the launch: cfg5 M=64 -> 1 4)
"""
import csv
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402

path, n, m = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
G, HB = (int(sys.argv[4]), int(sys.argv[5])) if len(sys.argv) > 5 else (1, 4)
piece = 64 - 2 * HB + 1
rows = [r for r in csv.reader(open(path)) if r]
hdr = next(r for r in rows if "Metric Name" in r)
ci, cv, ck = hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Kernel Name")
counts = [float(r[cv].replace(",", "")) for r in rows[rows.index(hdr) + 1:]
          if r[ci] == "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"]
X = synth.cfg5(n, m)
nnz = X.nnz.astype(np.int64)
live = np.arange(X.w)[None, :] < nnz[:, None]
ks = X.col[live]                                   # every step k of every row
P = int(nnz[ks].sum())                             # products
full, rest = nnz // piece, nnz % piece
steps = full * HB * ((piece + HB - 1) // HB) + HB * ((rest + HB - 1) // HB)  # steps incl. null padding
padded = int(64 * G * steps.sum())
assert int(nnz.max()) <= 64 * G
out = {"workload": f"cfg5 X^2 N={n} M={m}", "G": G, "HB": HB, "products": P, "steps": int(nnz.sum()),
       "steps_with_padding": int(steps.sum()), "predicted_dfma": padded, "ncu_dfma_per_launch": counts,
       "match": all(int(c) == padded for c in counts)}
print(json.dumps(out))
