import sys, numpy as np
sys.path.insert(0, '/root/repo')
from synth.planted import generate, tiny_spec
from tests.gpu_helpers import align, make_pair, rel_err
kw = dict(n=700, nnz=6000, d0=37, classes=5, clusters=14)
for prec in ["fp32", "bf16"]:
  for arch, dims, q in [("gcn", (37, 45, 29, 5), 3), ("sage", (23, 40, 33, 7), 4)]:
    g = generate(tiny_spec(**dict(kw, d0=dims[0], classes=dims[-1])), seed=0)
    gpu, ora = make_pair(g, arch, dims, optimizer="adam", q=q, precision=prec)
    gpu.partition(seed=99, m=2); ora.partition(seed=99, m=2)
    gpu.subtrain(1, lr=0.01)
    for i in range(2):
        ora.train_step(i, 0, 0.01)
        tr = ora.last_trace[i]
        nodes = gpu.trace(i, 0); p = align(nodes, tr["nodes"]); nb = len(nodes)
        lg = gpu.trace(i, 2).reshape(nb, -1); lo = tr["tape"]["logits"][p]
        bad = np.nonzero(np.abs(lg - lo).max(1) > 0.05 * np.abs(lo).max())[0]
        acts = [rel_err(gpu.trace(i, 1, l).reshape(nb, -1), tr["tape"]["H"][l][p]) for l in range(1, len(dims)-1)]
        print(prec, arch, "slot", i, "nb", nb, "logit err", rel_err(lg, lo), "bad rows", bad[:10], len(bad), "act errs", acts)
