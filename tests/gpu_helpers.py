"""Shared helpers of the -m gpu parity tests: build the same seeded problem on
the CUDA path (through the C ABI) and on the oracle, and compare per global
node id (the GPU orders batch rows by cluster; R14)."""
import numpy as np

from oracle import gist_oracle as O


def rel_err(x, r):
    """R18: normwise-max relative error max|x - r| / max|r|."""
    x = np.asarray(x, dtype=np.float64)
    r = np.asarray(r, dtype=np.float64)
    den = np.max(np.abs(r)) if r.size else 0.0
    if den == 0.0:
        return float(np.max(np.abs(x))) if x.size else 0.0
    return float(np.max(np.abs(x - r)) / den)


def make_pair(g, arch, dims, optimizer="adam", q=1, batch_seed=3, init_seed=7, precision="fp32"):
    from paper_2102_10424_b200.gist import Gist
    gpu = Gist(arch, dims, optimizer=optimizer, precision=precision, clusters_per_batch=q, batch_seed=batch_seed)
    gpu.load_graph(g)
    gpu.init_params(init_seed)
    ora = O.OracleGIST(arch=arch, dims=list(dims), optimizer=optimizer, clusters_per_batch=q, batch_seed=batch_seed)
    ora.load_graph(g["row_ptr"], g["col_idx"], g["X"], g["labels"], g["num_classes"], g["split"],
                   g["cluster_ids"], g["num_clusters"])
    ora.init_params(init_seed)
    return gpu, ora


def align(gpu_nodes, ora_nodes):
    """Index array p with ora_nodes[p] == gpu_nodes (same node set required)."""
    assert len(gpu_nodes) == len(ora_nodes)
    assert np.array_equal(np.sort(gpu_nodes), np.sort(ora_nodes))
    pos = {int(v): i for i, v in enumerate(ora_nodes)}
    return np.array([pos[int(v)] for v in gpu_nodes], dtype=np.int64)
