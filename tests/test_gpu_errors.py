"""The C ABI's state machine and argument checks (include/gist.h; SURVEY §8(b) "Errors"):
out-of-order calls return GIST_E_STATE, malformed graphs GIST_E_ARG / GIST_E_SHAPE, and a
failed call leaves the context usable (only CUDA / NCCL failures are sticky)."""
import numpy as np
import pytest

from synth.planted import generate, tiny_spec

pytestmark = pytest.mark.gpu


def small():
    return generate(tiny_spec(n=120, nnz=800, d0=6, classes=3, clusters=4), seed=0)


def ctx(**kw):
    from paper_2102_10424_b200.gist import Gist
    return Gist("gcn", (6, 8, 3), clusters_per_batch=2, **kw)


def test_state_machine():
    from paper_2102_10424_b200.gist import GistError
    g = small()
    c = ctx()
    with pytest.raises(GistError, match="STATE"):
        c.init_params(1)                       # no graph yet
    c.load_graph(g)
    with pytest.raises(GistError, match="STATE"):
        c.load_graph(g)                        # twice
    with pytest.raises(GistError, match="STATE"):
        c.partition(seed=1, m=2)               # no parameters
    c.set_params(0, np.zeros((6, 8), np.float32))
    with pytest.raises(GistError, match="STATE"):
        c.partition(seed=1, m=2)               # layer 1 never set
    c.set_params(1, np.zeros((8, 3), np.float32))
    c.partition(seed=1, m=2)                   # every layer set: PARAMS
    with pytest.raises(GistError, match="STATE"):
        c.partition(seed=2, m=2)               # twice without aggregate
    with pytest.raises(GistError, match="STATE"):
        c.eval(0)                              # open round
    with pytest.raises(GistError, match="STATE"):
        c.init_params(3)                       # open round
    c.subtrain(1, lr=0.1)
    c.aggregate()
    with pytest.raises(GistError, match="STATE"):
        c.aggregate()                          # no open round
    with pytest.raises(GistError, match="STATE"):
        c.subtrain(1, lr=0.1)                  # no partition
    c.eval(0)                                  # still usable after every refused call
    c.close()


def test_argument_errors():
    from paper_2102_10424_b200.gist import GistError
    c = ctx()
    c.load_graph(small())
    c.init_params(1)
    with pytest.raises(GistError, match="ARG"):
        c.partition(seed=1, m=0)
    with pytest.raises(GistError, match="ARG"):
        c.partition(seed=1, m=9)               # m > hidden dim 8
    with pytest.raises(GistError, match="ARG"):
        c.eval(4)                              # split code
    c.partition(seed=1, m=2)
    with pytest.raises(GistError, match="ARG"):
        c.subtrain(-1, lr=0.1)
    c.close()


def _mutate(g, fn):
    h = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in g.items()}
    fn(h)
    return h


def _drop_one_direction(h):
    """Remove one stored entry (u, v) but keep (v, u): the adjacency becomes asymmetric."""
    rp, ci = h["row_ptr"], h["col_idx"]
    u = int(np.argmax(np.diff(rp) > 0))
    e = rp[u]
    h["col_idx"] = np.delete(ci, e)
    h["row_ptr"] = np.concatenate([rp[:u + 1], rp[u + 1:] - 1])


def _duplicate_first_edge(h):
    rp, ci = h["row_ptr"], h["col_idx"]
    u = int(np.argmax(np.diff(rp) > 0))
    h["col_idx"] = np.insert(ci, rp[u], ci[rp[u]])
    h["row_ptr"] = np.concatenate([rp[:u + 1], rp[u + 1:] + 1])


def _unsort_row(h):
    rp, ci = h["row_ptr"], h["col_idx"]
    u = int(np.argmax(np.diff(rp) > 1))
    ci[rp[u]], ci[rp[u] + 1] = ci[rp[u] + 1], ci[rp[u]]


@pytest.mark.parametrize("name,fn,code", [
    ("asymmetric", _drop_one_direction, "ARG"),
    ("duplicate edge", _duplicate_first_edge, "ARG"),
    ("unsorted row", _unsort_row, "ARG"),
    ("col out of range", lambda h: h["col_idx"].__setitem__(0, h["n"] + 5), "ARG"),
    ("row_ptr decreasing", lambda h: h["row_ptr"].__setitem__(3, h["row_ptr"][4] + 1), "ARG"),
    ("label out of range", lambda h: h["labels"].__setitem__(0, 3), "ARG"),
    ("cluster id out of range", lambda h: h["cluster_ids"].__setitem__(0, 4), "ARG"),
    ("empty cluster", lambda h: h["cluster_ids"].__setitem__(h["cluster_ids"] == 2, 1), "ARG"),
    ("split code", lambda h: h["split"].__setitem__(0, 4), "ARG"),
    ("classes != d_L", lambda h: h.__setitem__("num_classes", 4), "SHAPE"),
])
def test_load_graph_rejects(name, fn, code):
    from paper_2102_10424_b200.gist import GistError
    g = _mutate(small(), fn)
    c = ctx()
    with pytest.raises(GistError, match=code):
        c.load_graph(g)
    c.load_graph(small())                      # the context stays usable
    c.close()


def test_q_larger_than_clusters():
    from paper_2102_10424_b200.gist import Gist, GistError
    c = Gist("gcn", (6, 8, 3), clusters_per_batch=5)
    with pytest.raises(GistError, match="ARG"):
        c.load_graph(small())
    c.close()
