import os, sys, numpy as np
pk = os.environ.get("PKGPATH", ".")
sys.path.insert(0, pk)
import paper_2506_03859_b200 as fqb
print("pkg", fqb.__file__)
from paper_2506_03859_b200 import FarpcaConfig, SketchKind, SketchSpec
rng = np.random.default_rng(7)
u,_ = np.linalg.qr(rng.standard_normal((600,120))); v,_ = np.linalg.qr(rng.standard_normal((400,120)))
a = np.asfortranarray((u*(0.95**np.arange(120)))@v.T)
for name, spec in (("stdbern-default", SketchSpec(SketchKind.StdBernoulli, 0.0, 3)),
                   ("stdbern-0.5", SketchSpec(SketchKind.StdBernoulli, 0.5, 3)),
                   ("bern-0.02", SketchSpec(SketchKind.Bernoulli, 0.02, 3)),
                   ("ssign", SketchSpec(SketchKind.SparseSign, 0.0, 3, zeta=8))):
    cfg = FarpcaConfig(eps=1e-2, power=1, block=16, sketch=spec, relative=True)
    es = [fqb.run_fixed_precision(a, cfg, output="host", svd=False).residual_sq for _ in range(4)]
    print(name, ["%.12e" % e for e in es], "DETERMINISTIC" if len(set(es)) == 1 else "VARIES")
