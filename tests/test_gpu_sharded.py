"""Site-block sharding on the GPU path: ranks emulated as threads of one process,
each block in its own C-ABI handle on cuda:0, exchanging device tensors through ThreadComm
(nothing on the device waits on another rank). Compared with a single handle over the whole
chain: identical bond profile and kept ranks, ledger and state equal up to FP reduction order
(the kernels' CTA shapes follow the wave's bucket, so the last bits of FP64 tail sums may
differ between a 1-rank and a 3-rank wave)."""
import threading

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _circuit():
    import workloads
    N, depth = 14, 9
    layers = workloads.brickwork_circuit(1, N, depth)
    kw = dict(d=2, f_min=0.99, n_planned=workloads.n_two_qubit_gates(layers), strategy="global")
    return N, layers, kw


@pytest.mark.parametrize("world", [2, 3])
def test_gpu_sharded_matches_single_handle(world):
    import paper_2307_16870_b200 as pk
    from paper_2307_16870_b200.sharded import GpuEngine, ShardedMPS, ThreadComm
    N, layers, kw = _circuit()
    ref = pk.MPS(N, slab_bytes=64 << 20, **kw)
    ref.run(layers)
    hub = ThreadComm.Hub(world)
    out, errs = {}, []

    def body(r):
        try:
            torch.cuda.set_device(0)
            sh = ShardedMPS(N, lambda n: GpuEngine(pk.MPS(n, slab_bytes=64 << 20, **kw)),
                            comm=ThreadComm(hub, r), device="cuda:0")
            sh.run(layers)
            out[r] = (sh.ledger(), sh.records(), sh.gather(0), sh.exchanges)
        except Exception as e:
            errs.append(e)
            raise

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    assert not errs, errs
    le, j, gu = out[0][0]
    e = ref.mps_fidelity_estimate()
    assert j == e["n_done"] and gu == int(e["guarantee_held"])
    assert abs(le - e["log_est"]) < 1e-9
    recs, rrecs = out[0][1], ref.mps_truncation_log()
    assert [(r["gate_index"], r["bond"], r["chi_before"], r["chi_after"]) for r in recs] == \
           [(r["gate_index"], r["bond"], r["chi_before"], r["chi_after"]) for r in rrecs]
    assert sum(o[3] for o in out.values()) > 0
    # gathered blocks -> a fresh single handle -> statevector overlap with the reference
    Bs, lams = out[0][2]
    g = pk.MPS(N, slab_bytes=64 << 20, **kw)
    g.mps_import_sites(0, [b.cpu().numpy() for b in Bs])
    s1, s2 = ref.mps_to_statevector(), g.mps_to_statevector()
    ov = abs(np.vdot(s1, s2)) ** 2 / (np.vdot(s1, s1).real * np.vdot(s2, s2).real)
    assert ov >= 1 - 1e-9, ov
    for b in range(N - 1):
        np.testing.assert_allclose(lams[b + 1].cpu().numpy(), ref.mps_schmidt_values(b), rtol=1e-5, atol=1e-7)
