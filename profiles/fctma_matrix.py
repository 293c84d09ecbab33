"""Run every (case, fc_tma config) of tests/test_gpu_parity.py::test_fc_tma_variants
in its own process (a crash does not poison the others); print ok / mismatch / crash."""
import itertools
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np, torch
from cases import case_inputs, oracle_outputs
from test_gpu_parity import run_on_gpu
from paper_1802_04730_b200 import ExecutionEngine
import conftest
from oracle_lib import Oracle
name, rows, cn, threads = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
golden = json.load(open("tests/golden/golden.json"))
oracle = Oracle()
ee = ExecutionEngine()
case, ins, seeded = case_inputs(oracle, golden, name)
o = {"block_shape": [1, 1, 1], "fusion_strategy": "max", "rng_seed": 0, "shared_memory_budget": 49152,
     "thread_shape": [threads, 1, 1], "tile_sizes": [rows, cn, 6], "unroll_copy_shared": False,
     "unroll_factor": 1, "use_private": False, "use_shared": True}
try:
    got, h = run_on_gpu(ee, case["def"], ins, seeded, options=o)
except Exception as e:
    print("SKIP/ERR", type(e).__name__, str(e)[:120]); sys.exit(0)
ref = oracle_outputs(oracle, case, ins, seeded)
bad = [k for k in ref if not np.array_equal(ref[k].view(np.uint32), got[k].view(np.uint32))]
print("MISMATCH " + ",".join(bad) if bad else "ok", ee.describe(h)["kernel"])
'''
cfgs = [(8, 8, 128), (4, 8, 64), (8, 4, 256), (3, 3, 96), (16, 8, 128), (1, 1, 64), (8, 16, 64), (8, 8, 64), (2, 2, 32)]
names = ["2fcrelu_small", "mlp3_small", "mlp3_paper", "mlp1_ragged", "mlp1_small", "2fcrelu_paper", "mlp1_paper"]
for (r, c, t), n in itertools.product(cfgs, names):
    p = subprocess.run([sys.executable, "-c", CHILD, n, str(r), str(c), str(t)], cwd=ROOT, capture_output=True,
                       text=True, timeout=120)
    out = (p.stdout.strip().splitlines() or [""])[-1]
    if p.returncode != 0:
        out = "CRASH rc=%d %s" % (p.returncode, (p.stderr.strip().splitlines() or [""])[-1][:100])
    print(f"{r:>3} {c:>3} {t:>4} {n:<14} {out}", flush=True)
