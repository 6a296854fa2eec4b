"""Model checkpoint file ("External Interfaces"): little-endian binary -- magic
"GIST", version u32, arch u8, L u32, dims u32[L+1], then every Theta_l row-major f32.  The
expected bytes are packed here with numpy from the oracle's parameters (tests/ only), never
from the CUDA path."""
import struct

import numpy as np
import pytest

import oracle.gist_oracle as O
from synth.planted import generate, tiny_spec
from tests.gpu_helpers import make_pair

pytestmark = pytest.mark.gpu
ARCH = {"gcn": 0, "sage": 1, "gat": 2}


def pack(arch, dims, theta):
    b = b"GIST" + struct.pack("<IBI", 1, ARCH[arch], len(dims) - 1)
    b += struct.pack(f"<{len(dims)}I", *dims)
    for w in theta:
        b += np.ascontiguousarray(w, dtype="<f4").tobytes()
    return b


def graph():
    return generate(tiny_spec(n=300, nnz=2400, d0=13, classes=4, clusters=6), seed=2)


@pytest.mark.parametrize("arch,dims", [("gcn", (13, 20, 4)), ("sage", (13, 17, 9, 4)), ("gat", (13, 24, 4))])
def test_save_matches_numpy_bytes(tmp_path, arch, dims):
    g = graph()
    gpu, ora = make_pair(g, arch, dims, q=2)
    theta = [np.asarray(t, dtype=np.float32) for t in ora.theta]
    for l, t in enumerate(theta):
        gpu.set_params(l, t)
    p = tmp_path / "m.gist"
    gpu.save_checkpoint(str(p))
    assert p.read_bytes() == pack(arch, dims, theta)


def test_load_then_train_round_trip(tmp_path):
    """A numpy-written file loads into a fresh context and trains like set_params would; a saved
    trained model reloads bit-identically (deterministic bytes)."""
    g = graph()
    dims = (13, 20, 4)
    a, ora = make_pair(g, "gcn", dims, q=2, optimizer="sgd")
    theta = [np.asarray(t, dtype=np.float32) for t in ora.theta]
    f = tmp_path / "init.gist"
    f.write_bytes(pack("gcn", dims, theta))
    b, _ = make_pair(g, "gcn", dims, q=2, optimizer="sgd")
    b.init_params(12345)                          # different weights, overwritten by the load
    b.load_checkpoint(str(f))
    for c in (a,):
        for l, t in enumerate(theta):
            c.set_params(l, t)
    for l in range(2):
        assert np.array_equal(b.get_params(l), theta[l])
    for c in (a, b):
        c.partition(seed=4, m=2)
        c.subtrain(3, lr=0.1)
        c.aggregate()
    fa, fb = tmp_path / "a.gist", tmp_path / "b.gist"
    a.save_checkpoint(str(fa))
    b.save_checkpoint(str(fb))
    assert fa.read_bytes() == fb.read_bytes()
    trained = [a.get_params(l) for l in range(2)]
    assert fa.read_bytes() == pack("gcn", dims, trained)
    c2, _ = make_pair(g, "gcn", dims, q=2)
    c2.load_checkpoint(str(fa))
    for l in range(2):
        assert np.array_equal(c2.get_params(l), trained[l])
    acc_a = a.eval(2)
    acc_c = c2.eval(2)
    assert acc_a == acc_c


def test_checkpoint_errors(tmp_path):
    from paper_2102_10424_b200.gist import Gist, GistError
    g = graph()
    dims = (13, 20, 4)
    gpu, ora = make_pair(g, "gcn", dims, q=2)
    good = pack("gcn", dims, ora.theta)
    cases = {
        "magic": (b"GISX" + good[4:], "ARG"),
        "version": (good[:4] + struct.pack("<I", 2) + good[8:], "ARG"),
        "arch": (good[:8] + bytes([1]) + good[9:], "SHAPE"),
        "dims": (pack("gcn", (13, 21, 4), [np.zeros((13, 21)), np.zeros((21, 4))]), "SHAPE"),
        "depth": (pack("gcn", (13, 20, 20, 4), [np.zeros((13, 20)), np.zeros((20, 20)), np.zeros((20, 4))]), "SHAPE"),
        "truncated": (good[:-3], "ARG"),
        "trailing": (good + b"\0", "ARG"),
        "header only": (good[:10], "ARG"),
    }
    for name, (blob, code) in cases.items():
        p = tmp_path / f"{name.replace(' ', '_')}.gist"
        p.write_bytes(blob)
        with pytest.raises(GistError, match=code):
            gpu.load_checkpoint(str(p))
    with pytest.raises(GistError, match="ARG"):
        gpu.load_checkpoint(str(tmp_path / "missing.gist"))
    with pytest.raises(GistError, match="ARG"):
        gpu.save_checkpoint(str(tmp_path / "no_such_dir" / "x.gist"))
    before = [gpu.get_params(l) for l in range(2)]        # refused loads changed nothing
    assert np.array_equal(before[0], np.asarray(ora.theta[0], np.float32))
    gpu.partition(seed=1, m=2)
    with pytest.raises(GistError, match="STATE"):
        gpu.save_checkpoint(str(tmp_path / "open.gist"))   # open round
    p = tmp_path / "ok.gist"
    p.write_bytes(good)
    with pytest.raises(GistError, match="STATE"):
        gpu.load_checkpoint(str(p))
    fresh = Gist("gcn", dims, clusters_per_batch=2)
    with pytest.raises(GistError, match="STATE"):
        fresh.load_checkpoint(str(p))                     # no graph yet
    fresh.load_graph(g)
    fresh.load_checkpoint(str(p))                         # graph -> PARAMS
    fresh.partition(seed=1, m=2)
    fresh.close()
