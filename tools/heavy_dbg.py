import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np
from tests.test_gpu_heavy_rows import hub_graph
from tests.gpu_helpers import align, make_pair, rel_err
arch, dims = sys.argv[1], tuple(int(x) for x in sys.argv[2].split(','))
g = hub_graph()
gpu, ora = make_pair(g, arch, dims, optimizer="adam", q=2, precision=sys.argv[3])
gpu.partition(seed=7, m=2); ora.partition(seed=7, m=2)
gpu.subtrain(1, lr=0.01)
out = []
for i in range(2):
    ora.train_step(i, 0, 0.01)
    tr = ora.last_trace[i]
    nodes = gpu.trace(i, 0); p = align(nodes, tr["nodes"]); nb = len(nodes)
    e = [rel_err(gpu.trace(i, 2).reshape(nb, -1), tr["tape"]["logits"][p])]
    e += [rel_err(gpu.trace(i, 1, l).reshape(nb, -1), tr["tape"]["H"][l][p]) for l in range(1, len(dims) - 1)]
    e += [rel_err(gpu.trace(i, 3, l).reshape(ora.sub[i][l].shape), tr["grads"][l]) for l in range(len(dims) - 1)]
    out.append(["%.2e" % x for x in e])
print(arch, dims, sys.argv[3], {k: v for k, v in os.environ.items() if k.startswith('GIST_')}, out, flush=True)
