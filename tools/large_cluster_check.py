"""Weight error of the large-cluster BF16 case (clusters of ~200 rows) under each aggregation path."""
import os, sys, json
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from synth.planted import generate, tiny_spec
from tests.gpu_helpers import make_pair, rel_err
g = generate(tiny_spec(n=1000, nnz=24000, d0=36, classes=5, clusters=5, f_in=0.8), seed=6)
out = {"env": {k: v for k, v in os.environ.items() if k.startswith("GIST_")}}
for prec in ("bf16", "fp32"):
    gpu, ora = make_pair(g, "sage", (36, 80, 5), optimizer="sgd", q=2, precision=prec)
    errs = []
    for t in range(2):
        gpu.partition(seed=9 + t, m=2); ora.partition(seed=9 + t, m=2)
        lg = gpu.subtrain(4, lr=0.1); lo = ora.subtrain(4, lr=0.1)
        gpu.aggregate(); ora.aggregate()
        errs.append([float(rel_err(gpu.get_params(l), ora.theta[l])) for l in range(2)] + [float(np.max(np.abs(lg - lo)))])
    out[prec] = errs
print(json.dumps(out))
