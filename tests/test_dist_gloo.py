"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 subAgg protocol
(PAPER.md:140, 169, 185-190):
  * slot i lives on rank gist_slot_owner(i, W) (the library's own layout functions);
  * every rank derives the same partition from the counter-based PRNG (no exchange);
  * one all-gather of equal-size packed slot buffers per round, then every rank writes
    all m blocks into its replica.
The sub-GCN arithmetic runs in the FP64 oracle here (the test engine); the transport is
torch.distributed gloo.  Property: the global Theta after every round is bit-identical to
the single-process run and across ranks (world-size invariance)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import gist_oracle as O
from synth.planted import generate, tiny_spec

DIMS = (12, 20, 15, 4)
M, ROUNDS, ZETA = 3, 2, 3


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def make(opt_state="reset", arch="sage"):
    g = generate(tiny_spec(n=240, nnz=1500, d0=12, classes=4, clusters=8), seed=3)
    o = O.OracleGIST(arch=arch, dims=list(DIMS), optimizer="adam", clusters_per_batch=2, batch_seed=9,
                     opt_state=opt_state)
    o.load_graph(g["row_ptr"], g["col_idx"], g["X"], g["labels"], g["num_classes"], g["split"],
                 g["cluster_ids"], g["num_clusters"])
    o.init_params(5)
    return o


def pack(subs, slots, spr, smax):
    buf = np.zeros(spr * smax)
    for j, i in enumerate(slots):
        flat = np.concatenate([w.ravel() for w in subs[i]])
        buf[j * smax: j * smax + len(flat)] = flat
    return buf


def unpack(flat, shapes):
    out, off = [], 0
    for s in shapes:
        n = s[0] * s[1]
        out.append(flat[off: off + n].reshape(s))
        off += n
    return out


def p2p_exchange(rank, world, blocks_of, apply):
    """agg_mode P2P as gist_aggregate runs it: barrier; each owner stores its
    own slots i = rank, rank + W, ... (i // W = local index) into every rank's replica; barrier.
    A peer store is a point-to-point send here (gloo has no peer memory); the oracle is FP64,
    and the copy is bitwise either way (R9)."""
    dist.barrier()
    own = list(range(rank, M, world))
    reqs = []
    for i in own:
        buf = torch.from_numpy(np.ascontiguousarray(blocks_of(i), dtype=np.float64))
        apply(i, buf.numpy())                               # the local replica
        reqs += [dist.isend(buf, dst=r, tag=i) for r in range(world) if r != rank]
    for i in range(M):
        if i in own:
            continue
        buf = torch.zeros(blocks_of(i).size, dtype=torch.float64)
        dist.recv(buf, src=i % world, tag=i)                # owner = gist_slot_owner(i, W)
        apply(i, buf.numpy())
    for r in reqs:
        r.wait()
    dist.barrier()


def sharded_run(rank, world, opt_state="reset", arch="sage", transport="allgather"):
    from paper_2102_10424_b200 import gist
    o = make(opt_state, arch)
    spr = gist.slots_per_rank(M, world)
    mine = gist.local_slots(M, world, rank)
    history = []
    for t in range(ROUNDS):
        o.partition(seed=77, m=M)                     # identical on every rank (Philox, no exchange)
        shapes = [[w.shape for w in o.sub[i]] for i in range(M)]
        smax = max(sum(a * b for a, b in s) for s in shapes)
        for i in mine:                                # subTrain only the local slots
            for z in range(ZETA):
                o.train_step(i, o.step + z, 0.01)
        o.step += ZETA
        # the one exchange of the round: the packed slot weights (and, with persistent Adam
        # state, the two moment slices the same way)
        tensors = [("w", o.sub)]
        if opt_state == "persistent":
            tensors += [(k, [[st[k] for st in so] for so in o.opt]) for k in ("m", "v")]
        for name, blocks in tensors:
            if transport == "p2p":
                def blocks_of(i, blocks=blocks):
                    return np.concatenate([b.ravel() for b in blocks[i]])

                def apply(i, flat, name=name):
                    got = unpack(flat, shapes[i])
                    if name == "w":
                        o.sub[i] = got
                    else:
                        for l in range(len(got)):
                            o.opt[i][l][name] = got[l]
                            o.opt[i][l]["t"] = o.t_global + ZETA
                p2p_exchange(rank, world, blocks_of, apply)
                continue
            send = torch.from_numpy(pack(blocks, mine, spr, smax))
            recv = [torch.zeros_like(send) for _ in range(world)]
            dist.all_gather(recv, send)
            for r in range(world):
                for j in range(spr):
                    i = r + world * j
                    if i >= M:
                        continue
                    assert gist.slot_owner(i, world) == r
                    got = unpack(recv[r].numpy()[j * smax:(j + 1) * smax], shapes[i])
                    if name == "w":
                        o.sub[i] = got
                    else:
                        for l in range(len(got)):
                            o.opt[i][l][name] = got[l]
                            o.opt[i][l]["t"] = o.t_global + ZETA   # every slot took ZETA steps
        o.aggregate()
        history.append([w.copy() for w in o.theta] +
                       ([m.copy() for m in o.mom] + [v.copy() for v in o.vel] if opt_state == "persistent" else []))
    return history


def worker(rank, world, port, q, opt_state="reset", arch="sage", transport="allgather"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        hist = sharded_run(rank, world, opt_state, arch, transport)
        q.put((rank, [[w.tobytes() for w in th] for th in hist]))
    finally:
        dist.destroy_process_group()


def reference(opt_state="reset", arch="sage"):
    o = make(opt_state, arch)
    hist = []
    for t in range(ROUNDS):
        o.partition(seed=77, m=M)
        o.subtrain(ZETA, 0.01)
        o.aggregate()
        hist.append([w.copy() for w in o.theta] +
                    ([m.copy() for m in o.mom] + [v.copy() for v in o.vel] if opt_state == "persistent" else []))
    return hist


def test_layout_functions():
    from paper_2102_10424_b200 import gist
    for m in (1, 2, 3, 8, 13):
        for W in (1, 2, 4, 8):
            owners = [gist.slot_owner(i, W) for i in range(m)]
            assert owners == [i % W for i in range(m)]
            assert gist.slots_per_rank(m, W) == -(-m // W)
            assert sorted(sum((gist.local_slots(m, W, r) for r in range(W)), [])) == list(range(m))


@pytest.mark.timeout(300)
@pytest.mark.parametrize("opt_state,arch,transport", [("reset", "sage", "allgather"), ("persistent", "sage", "allgather"),
                                                      ("reset", "gat", "allgather"), ("reset", "sage", "p2p"),
                                                      ("persistent", "sage", "p2p")])
def test_world2_gloo_bit_identical_to_world1(opt_state, arch, transport):
    """(GAT, R21: the last layer's attention rows are the mean of all m copies, so every rank
    needs every slot's copy -- the same all-gather delivers them; agg_mode P2P refuses GAT.)"""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, q, opt_state, arch, transport)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = reference(opt_state, arch)
    for t in range(ROUNDS):
        assert len(ref[t]) == len(res[0][t]) == (len(DIMS) - 1) * (3 if opt_state == "persistent" else 1)
        for l in range(len(ref[t])):        # weights (and global moments) per layer
            want = ref[t][l].tobytes()
            assert res[0][t][l] == want and res[1][t][l] == want, (t, l)


def eval_worker(rank, world, port, q):
    """Partition-wise eval protocol of gist_eval_parts for world > 1 (R20): rank r evaluates the
    partitions p with p mod W == r, the per-partition (CE sum, correct, count) triples are summed
    across ranks (the library's one ncclAllReduce; gloo here), every rank averages."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        o = make()
        n = len(o.labels)
        part = (np.arange(n) * 5) % 7
        mine = [p for p in range(7) if p % world == rank]
        _, _, lp, ap = o.eval_partitions(0, part, 7, parts=mine)
        sums = np.zeros((7, 3))
        for p in mine:
            cnt = float(np.sum((part == p) & (o.split == 0)))
            if cnt:
                sums[p] = [lp[p] * cnt, ap[p] * cnt, cnt]
        t = torch.from_numpy(sums)
        dist.all_reduce(t)
        s = t.numpy()
        ok = s[:, 2] > 0
        q.put((rank, float(np.mean(s[ok, 0] / s[ok, 2])), float(np.mean(s[ok, 1] / s[ok, 2]))))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_world2_gloo_partition_eval_protocol():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=eval_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (l, a)) for r, l, a in (q.get(timeout=240) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    o = make()
    n = len(o.labels)
    lw, aw, _, _ = o.eval_partitions(0, (np.arange(n) * 5) % 7, 7)
    for r in (0, 1):
        assert res[r][0] == pytest.approx(lw, rel=1e-12) and res[r][1] == pytest.approx(aw, rel=1e-12)
