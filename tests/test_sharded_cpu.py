"""Site-block sharding on CPU: gloo, world sizes 2 and 3.

The host logic of paper_2307_16870_b200/sharded.py (partition, ghost fetch, boundary
write-back, ledger token chain, gather) drives an engine; here the engine is the complex128
oracle (test infrastructure), so every gate update is computed exactly as in a single-handle run
and the sharded result must be BIT-IDENTICAL to world 1 ("bit-identical output to
world 1"): bond profile, ledger (log E, j, guarantee), every truncation record, every site
tensor and Schmidt vector, and the gathered state's amplitudes.
"""
import os
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class OracleEngine:
    """Engine interface of ShardedMPS over oracle.OracleMPS (complex128 numpy <-> CPU tensors)."""

    def __init__(self, n_local, **kw):
        import oracle
        self.o = oracle.OracleMPS(n_local, **kw)
        self.pending = None

    def layer_begin(self, sites, Us):
        self.pending = (np.asarray(sites, np.int32), np.asarray(Us))
        return 1

    def layer_step(self):
        s, u = self.pending
        self.pending = None
        self.o.apply_layer(s, u)
        return 0

    def ledger_get(self):
        e = self.o.estimate()
        return e["log_est"], e["n_done"], int(e["guarantee_held"])

    def ledger_set(self, log_E, j, guarantee):
        self.o.set_ledger(log_E, j, guarantee)

    def export_site(self, site):
        return torch.from_numpy(self.o.export_site(site))

    def import_site(self, site, B):
        self.o.import_site(site, B.numpy())

    def get_lambda(self, bond):
        return torch.from_numpy(self.o.schmidt_values(bond))

    def set_lambda(self, bond, lam):
        self.o.set_lambda(bond, lam.numpy())

    def records(self):
        return self.o.records()


def _circuit(kind):
    import workloads
    if kind == "mps":
        N, depth = 14, 9
        layers = workloads.brickwork_circuit(1, N, depth)
        kw = dict(d=2, f_min=0.99, n_planned=workloads.n_two_qubit_gates(layers), strategy="global")
    else:
        N, depth = 10, 5
        layers = workloads.mpo_circuit(4, N, depth, 0.01)
        kw = dict(d=4, f_min=0.95, n_planned=workloads.n_two_qubit_gates(layers), strategy="nearest",
                  rule="wang")
    return N, layers, kw


def _worker(rank, world, port, kind, out):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2307_16870_b200.sharded import ShardedMPS
        N, layers, kw = _circuit(kind)
        sh = ShardedMPS(N, lambda n: OracleEngine(n, **kw), cdtype=torch.complex128, rdtype=torch.float64)
        sh.run(layers)
        recs = sh.records()
        led = sh.ledger()
        g = sh.gather(0)
        if rank == 0:
            Bs, lams = g
            out.put(("ok", rank, dict(ledger=led, records=recs, B=[b.numpy() for b in Bs],
                                      lam=[l.numpy() for l in lams], blocks=sh.blocks, ex=sh.exchanges)))
        else:
            out.put(("ok", rank, dict(ledger=led, ex=sh.exchanges)))
        dist.barrier()
    except Exception as e:  # surface the failure in the parent
        import traceback
        out.put(("err", rank, traceback.format_exc()))
        raise
    finally:
        dist.destroy_process_group()


def _run(world, kind):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29000 + (os.getpid() * 7 + world * 101 + (kind == "mpo") * 13) % 2000
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        st, r, payload = q.get(timeout=300)
        assert st == "ok", payload
        res[r] = payload
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def _reference(kind):
    import oracle
    N, layers, kw = _circuit(kind)
    o = oracle.OracleMPS(N, **kw)
    o.run(layers)
    return N, o


def test_partition_even_boundaries():
    from paper_2307_16870_b200.sharded import partition
    for N, p in [(12, 2), (14, 3), (300, 8), (300, 7), (50, 4), (16, 8)]:
        blocks = partition(N, p)
        assert blocks[0][0] == 0 and blocks[-1][1] == N
        for (a, b), (c, _) in zip(blocks[:-1], blocks[1:]):
            assert b == c and b % 2 == 0 and b - a >= 2
    # cost-weighted: heavy middle sites pull the boundaries inwards
    w = np.ones(40)
    w[10:30] = 100.0
    blocks = partition(40, 2, w)
    assert blocks[0][1] == 20
    with pytest.raises(ValueError):
        partition(3, 2)


@pytest.mark.parametrize("world,kind", [(2, "mps"), (3, "mps"), (2, "mpo")])
def test_sharded_bit_identical_to_world1(world, kind):
    N, ref = _reference(kind)
    res = _run(world, kind)
    r0 = res[0]
    e = ref.estimate()
    for r in range(world):   # every rank ends with the same token == the single-handle ledger
        assert res[r]["ledger"] == (e["log_est"], e["n_done"], int(e["guarantee_held"]))
    assert r0["records"] == ref.records()
    for i in range(N):
        np.testing.assert_array_equal(r0["B"][i], ref.export_site(i))
    for b in range(-1, N):
        np.testing.assert_array_equal(r0["lam"][b + 1], ref.schmidt_values(b))
    # the boundary exchange happened (odd layers straddle every boundary)
    assert sum(res[r]["ex"] for r in range(world)) > 0
    # gathered state -> a fresh single handle -> same amplitudes
    import oracle
    _, _, kw = _circuit(kind)
    o2 = oracle.OracleMPS(N, **kw)
    for i in range(N):
        o2.import_site(i, r0["B"][i])
    rng = np.random.default_rng(7)
    for _ in range(5):
        dg = rng.integers(0, kw["d"], N).astype(np.uint8)
        assert o2.amplitude(dg) == ref.amplitude(dg)


def test_thread_ranks_match_world1():
    """The in-process transport (ranks as threads, as the one-GPU test uses) gives the same
    bit-identical result as the gloo ranks."""
    import threading

    from paper_2307_16870_b200.sharded import ShardedMPS, ThreadComm
    N, ref = _reference("mps")
    _, layers, kw = _circuit("mps")
    world = 3
    hub = ThreadComm.Hub(world)
    out, errs = {}, []

    def body(r):
        try:
            sh = ShardedMPS(N, lambda n: OracleEngine(n, **kw), comm=ThreadComm(hub, r),
                            cdtype=torch.complex128, rdtype=torch.float64)
            sh.run(layers)
            out[r] = (sh.ledger(), sh.records(), sh.gather(0))
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)
            raise

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    assert not errs, errs
    e = ref.estimate()
    assert out[0][0] == (e["log_est"], e["n_done"], int(e["guarantee_held"]))
    assert out[0][1] == ref.records()
    Bs, _ = out[0][2]
    for i in range(N):
        np.testing.assert_array_equal(Bs[i].numpy(), ref.export_site(i))
