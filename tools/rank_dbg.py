import json, sys, math
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from oracle.oracle import Oracle
from paper_2506_03859_b200 import experiment as ex
from test_experiment import GRID_RANK
import tempfile, os
d = tempfile.mkdtemp()
ref = Oracle("reference")
p = os.path.join(d, "c.json"); json.dump(dict(GRID_RANK, out_prefix=os.path.join(d, "ref")), open(p, "w"))
assert ref.run_experiment(p) is None
r = ex.read_report_csv(os.path.join(d, "ref.csv"))
cfg = ex.load_experiment_config(p); cfg.out_prefix = os.path.join(d, "ours")
rep = ex.run_experiment(cfg)
for g, q in zip(rep.records, r):
    flag = "" if abs(g.err - q.err) < 1e-9 else "  <-- DIFF"
    print(g.algorithm, g.power, g.l, g.r, f"{g.err:.6g} {q.err:.6g}", g.note[:40], flag)
