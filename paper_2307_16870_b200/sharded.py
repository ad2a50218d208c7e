"""Multi-GPU site-block sharding of one long MPS.

One process per GPU; rank g owns the contiguous block of sites [lo_g, hi_g) with every boundary
lo_g even, so that the gates of an even layer (pairs (2j, 2j+1)) never straddle a boundary and
an odd layer straddles each boundary exactly once, at the pair (hi_g - 1, hi_g). The B-lambda
(Vidal/Hastings) form makes the gates of a layer independent (PAPER.md:114 contracts only the
two neighbouring tensors; the canonical form PAPER.md:84, 142 is the B-lambda reading of
DESIGN.md), so the only exchange steps are:

  * ghost fetch (before a layer that holds the boundary gate): rank g+1 sends its first site
    tensor B_{hi_g} to rank g, which keeps it as an extra local "ghost" site;
  * boundary write-back (after that layer): rank g sends the new B_{hi_g} = V_k^H and the new
    Schmidt vector lambda_{hi_g - 1} to rank g+1;
  * ledger token: the truncation targets of the global/nearest strategies depend on the running
    product E of all previous truncation fidelities in canonical order (E12/E14, PAPER.md:132-148;
    DESIGN.md reading 5: layer-major, ascending site). Rank g's select waits for (log E, j) from
    rank g-1 -- the contractions and SVDs of all ranks run concurrently (mps_layer_begin) -- and
    the last rank broadcasts the end-of-layer token.

Results are therefore bit-identical to a single handle over the whole chain (same kernels, same
inputs per gate, same ledger order). The transport is torch.distributed point-to-point (NCCL
over NVLink on GPUs, gloo in the CPU tests); every gate update still runs in the engine -- the
CUDA library through its C ABI (GpuEngine) or, in the tests only, any object with the same
methods.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def partition(n_sites: int, world: int, weights=None):
    """Contiguous blocks [lo_g, hi_g) with even interior boundaries, balanced by the per-site
    cost `weights` (default uniform; DESIGN.md suggests the predicted sum of chi^3)."""
    if world < 1 or n_sites < 2 * world:
        raise ValueError("need at least two sites per rank")
    w = np.ones(n_sites) if weights is None else np.asarray(weights, np.float64)
    cum = np.concatenate([[0.0], np.cumsum(w)])
    cuts = [0]
    for g in range(1, world):
        target = cum[-1] * g / world
        b = int(np.searchsorted(cum, target))
        b = max(cuts[-1] + 2, min(b + (b & 1), n_sites - 2 * (world - g)))
        b += b & 1
        cuts.append(b)
    cuts.append(n_sites)
    for a, b in zip(cuts[:-1], cuts[1:]):
        if b - a < 2:
            raise ValueError("partition failed: %s" % cuts)
    return [(cuts[g], cuts[g + 1]) for g in range(world)]


def predicted_site_cost(n_sites: int, depth: int, d: int = 2, chi_cap: int = 0):
    """Per-site cost model for partition(): the predicted sum over the run of chi^3 at the site's
    right bond (the SVD of a theta with chi_l ~ chi_r ~ chi costs ~chi^3). chi of bond
    b after t brickwork layers is bounded by the rank bound min(d^(t+1), d^(b+1), d^(N-1-b)) (the
    bulk grows by d per layer from the product state, the chain ends are limited by the Hilbert
    space of the shorter side, SURVEY §8(d) "rank bound"), capped at chi_cap. The ~12 edge sites
    of a 300-site chain stay far below the bulk, so uniform blocks underload the edge ranks."""
    cost = np.zeros(n_sites)
    for b in range(n_sites):
        edge = min(b + 1, n_sites - 1 - b)
        tot = 0.0
        for t in range(depth):
            e = float(min(t + 1, edge))
            chi = d ** min(e, 60.0)
            if chi_cap > 0:
                chi = min(chi, float(chi_cap))
            tot += chi ** 3
        cost[b] = max(tot, 1.0)
    return cost


class GpuEngine:
    """Adapter of the C-ABI binding (MPS) to the engine interface of ShardedMPS (device tensors)."""

    def __init__(self, mps):
        self.m = mps
        self.device = mps.device

    def layer_begin(self, sites, Us):
        return self.m.mps_layer_begin(sites, Us)

    def layer_step(self):
        return self.m.mps_layer_step()

    def ledger_get(self):
        return self.m.mps_ledger_get()

    def ledger_set(self, log_E, j, guarantee):
        self.m.mps_ledger_set(log_E, j, guarantee)

    def export_site(self, site):
        from . import C, _ptr, lib
        dims = np.zeros(3, np.int32)
        self.m._check(lib().mps_export_site(self.m._h, int(site), None, _ptr(dims)))
        B = torch.empty(tuple(int(x) for x in dims), dtype=torch.complex64, device=self.device)
        self.m._check(lib().mps_export_site(self.m._h, int(site), C.c_void_p(B.data_ptr()), _ptr(dims)))
        return B

    def import_site(self, site, B):
        self.m.mps_import_site(site, B.to(self.device, torch.complex64).contiguous())

    def get_lambda(self, bond):
        from . import C, _ptr, lib
        ln = C.c_int32(0)
        self.m._check(lib().mps_schmidt_values(self.m._h, int(bond), None, 0, C.byref(ln)))
        lam = torch.empty(ln.value, dtype=torch.float32, device=self.device)
        self.m._check(lib().mps_schmidt_values(self.m._h, int(bond), C.c_void_p(lam.data_ptr()), ln.value,
                                               C.byref(ln)))
        return lam

    def set_lambda(self, bond, lam):
        from . import C, lib
        lam = lam.to(self.device, torch.float32).contiguous()
        self.m._check(lib().mps_set_lambda(self.m._h, int(bond), C.c_void_p(lam.data_ptr()), int(lam.numel())))

    def records(self):
        return self.m.mps_truncation_log()


class DistComm:
    """torch.distributed point-to-point transport (NCCL on GPUs, gloo on CPU)."""

    def __init__(self):
        self.rank, self.world = dist.get_rank(), dist.get_world_size()

    def send(self, t: torch.Tensor, dst: int):
        shape = torch.tensor(list(t.shape) + [-1] * (4 - t.dim()), dtype=torch.int64, device=t.device)
        dist.send(shape, dst)
        dist.send(torch.view_as_real(t).contiguous() if t.is_complex() else t.contiguous(), dst)

    def recv(self, src: int, dtype, device) -> torch.Tensor:
        shape = torch.empty(4, dtype=torch.int64, device=device)
        dist.recv(shape, src)
        dims = [int(x) for x in shape.tolist() if x >= 0]
        if dtype.is_complex:
            real = torch.float32 if dtype == torch.complex64 else torch.float64
            buf = torch.empty(dims + [2], dtype=real, device=device)
            dist.recv(buf, src)
            return torch.view_as_complex(buf)
        buf = torch.empty(dims, dtype=dtype, device=device)
        dist.recv(buf, src)
        return buf

    def broadcast(self, t: torch.Tensor, src: int):
        dist.broadcast(t, src=src)
        return t

    def all_gather_object(self, obj):
        out = [None] * self.world
        dist.all_gather_object(out, obj)
        return out


class ThreadComm:
    """In-process transport for ranks run as threads of one process (tests: several blocks on
    ONE GPU, each with its own handle; nothing on the device waits on another rank)."""

    class Hub:
        def __init__(self, world):
            import queue
            self.world = world
            self.q = [[queue.Queue() for _ in range(world)] for _ in range(world)]

    def __init__(self, hub, rank):
        self.hub, self.rank, self.world = hub, rank, hub.world

    def send(self, t, dst):
        self.hub.q[self.rank][dst].put(t.clone())

    def recv(self, src, dtype, device):
        t = self.hub.q[src][self.rank].get(timeout=600)
        assert t.dtype == dtype, (t.dtype, dtype)
        return t.to(device)

    def broadcast(self, t, src):
        if self.rank == src:
            for r in range(self.world):
                if r != src:
                    self.hub.q[src][r].put(t.clone())
            return t
        t.copy_(self.hub.q[src][self.rank].get(timeout=600))
        return t

    def all_gather_object(self, obj):
        for r in range(self.world):
            if r != self.rank:
                self.hub.q[self.rank][r].put(obj)
        return [obj if r == self.rank else self.hub.q[r][self.rank].get(timeout=600) for r in range(self.world)]


class ShardedMPS:
    """One rank's block of a site-sharded EA-MPS/MPO.

    engine_factory(n_local) must return an engine (GpuEngine, or a test double) holding
    n_local = (hi - lo) + ghost sites in the product state |0...0>; `ghost` = 1 on every rank
    but the last. Local site x is global site lo + x; local bond b is global bond lo + b.
    """

    def __init__(self, n_sites: int, engine_factory, comm=None, blocks=None, device=None,
                 cdtype=torch.complex64, rdtype=torch.float32, weights=None):
        """comm: DistComm() (default when torch.distributed is initialised), ThreadComm, or None
        for a single block (world 1). blocks: explicit [lo, hi) per rank, else partition() by
        `weights` (e.g. predicted_site_cost; default uniform)."""
        if comm is None and dist.is_available() and dist.is_initialized():
            comm = DistComm()
        self.comm = comm
        self.rank = comm.rank if comm is not None else 0
        self.world = comm.world if comm is not None else 1
        self.N = n_sites
        self.blocks = partition(n_sites, self.world, weights) if blocks is None else list(blocks)
        self.lo, self.hi = self.blocks[self.rank]
        self.ghost = 1 if self.rank < self.world - 1 else 0
        self.eng = engine_factory(self.hi - self.lo + self.ghost)
        self.device = torch.device("cpu") if device is None else torch.device(device)
        self.cdtype, self.rdtype = cdtype, rdtype
        # ghost bookkeeping, updated identically on both sides of a boundary from the (global) layer:
        # our ghost copy of B_hi is stale <=> rank g+1's first site changed since the last fetch
        self.ghost_stale = True
        self._first_dirty = True
        self.exchanges = 0         # boundary messages this rank sent (for tests / bench)

    # ---- helpers -----------------------------------------------------------------------------
    def _crossing(self, g, sites):
        """Does the layer hold the boundary gate (hi_g - 1, hi_g) of rank g?"""
        return g < self.world - 1 and (self.blocks[g][1] - 1) in sites

    def _touches_first(self, g, sites):
        """Does the layer hold a gate on rank g's first site (lo_g, lo_g + 1)?"""
        return g > 0 and self.blocks[g][0] in sites

    def _token(self, vals):
        return torch.tensor(vals, dtype=torch.float64, device=self.device)

    # ---- one brickwork layer -----------------------------------------------------------------
    def apply_layer(self, sites, Us):
        """Apply one layer of disjoint gates given GLOBALLY (every rank passes the same layer)."""
        sites = np.asarray(sites, np.int64).ravel()
        Us = np.asarray(Us)
        S = set(int(x) for x in sites)
        g, p = self.rank, self.world
        # a6 (1): ghost fetch. Rank g+1 sends its first site to rank g when the layer crosses the
        # boundary g|g+1 and that site changed since the last fetch (both sides track this).
        if p > 1:
            send_first = g > 0 and self._crossing(g - 1, S) and self._first_dirty
            recv_ghost = self._crossing(g, S) and self.ghost_stale
            # even ranks send first, odd ranks receive first: no cycle of blocking sends
            ops = [("s", send_first), ("r", recv_ghost)]
            if g % 2:
                ops.reverse()
            for kind, on in ops:
                if not on:
                    continue
                if kind == "s":
                    self.comm.send(self.eng.export_site(0).to(self.device), g - 1)
                    self._first_dirty = False
                    self.exchanges += 1
                else:
                    B = self.comm.recv(g + 1, self.cdtype, self.device)
                    self.eng.import_site(self.hi - self.lo, B)
                    self.ghost_stale = False
        # local gates (global i in [lo, hi); i = hi - 1 pairs with the ghost)
        mine = [x for x in range(sites.size) if self.lo <= sites[x] < self.hi]
        loc_sites = np.array([sites[x] - self.lo for x in mine], np.int32)
        loc_us = Us[mine] if mine else Us[:0]
        waves = self.eng.layer_begin(loc_sites, loc_us) if mine else 0   # a0-a3, not waited on
        # ledger token chain (canonical order = ascending global site = rank order)
        if g > 0:
            tok = self.comm.recv(g - 1, torch.float64, self.device).tolist()
            self.eng.ledger_set(tok[0], int(tok[1]), int(tok[2]))
        if waves:
            while self.eng.layer_step() > 0:
                pass
        le, j, gu = self.eng.ledger_get()
        if g < p - 1:
            self.comm.send(self._token([le, float(j), float(gu)]), g + 1)
        final = self._token([le, float(j), float(gu)])
        if p > 1:
            self.comm.broadcast(final, p - 1)
            fl = final.tolist()
            if g < p - 1:
                self.eng.ledger_set(fl[0], int(fl[1]), int(fl[2]))
        # a6 (2): boundary write-back. Rank g sends the new B_hi and lambda_{hi-1} to rank g+1.
        if p > 1:
            send_back = self._crossing(g, S)
            recv_back = g > 0 and self._crossing(g - 1, S)
            ops = [("s", send_back), ("r", recv_back)]
            if g % 2:
                ops.reverse()
            for kind, on in ops:
                if not on:
                    continue
                if kind == "s":
                    gl = self.hi - self.lo
                    self.comm.send(self.eng.export_site(gl).to(self.device), g + 1)
                    self.comm.send(self.eng.get_lambda(gl - 1).to(self.device), g + 1)
                    self.exchanges += 1
                else:
                    B = self.comm.recv(g - 1, self.cdtype, self.device)
                    lam = self.comm.recv(g - 1, self.rdtype, self.device)
                    self.eng.import_site(0, B)
                    self.eng.set_lambda(-1, lam)
            # a gate on rank g's first site makes rank g-1's ghost stale (the boundary write-back
            # leaves both copies equal, so it does not)
            if g > 0 and self._touches_first(g, S):
                self._first_dirty = True
            if g < p - 1 and self._touches_first(g + 1, S):
                self.ghost_stale = True

    def run(self, layers):
        for sites, us in layers:
            self.apply_layer(sites, us)

    # ---- queries -----------------------------------------------------------------------------
    def ledger(self):
        return self.eng.ledger_get()

    def records(self):
        """All ranks' truncation records in canonical (gate_index) order, on every rank."""
        mine = [dict(r, bond=r["bond"] + self.lo) for r in self.eng.records()]   # local -> global bond
        if self.world == 1:
            return mine
        allr = self.comm.all_gather_object(mine)
        return sorted([r for rs in allr for r in rs], key=lambda r: r["gate_index"])

    def gather(self, dst: int = 0):
        """Owned site tensors and Schmidt vectors of the whole chain on rank `dst`:
        returns (list of N site tensors, list of N+1 lambdas for bonds -1..N-1) there, None elsewhere."""
        own = self.hi - self.lo
        Bs = [self.eng.export_site(x).to(self.device) for x in range(own)]
        lams = [self.eng.get_lambda(b).to(self.device) for b in range(-1 if self.rank == 0 else 0, own)]
        if self.world == 1:
            return Bs, lams
        if self.rank != dst:
            for t in Bs:
                self.comm.send(t, dst)
            for t in lams:
                self.comm.send(t, dst)
            return None
        out_B, out_l = [None] * self.N, [None] * (self.N + 1)
        for g in range(self.world):
            lo, hi = self.blocks[g]
            if g == dst:
                gB, gl = Bs, lams
            else:
                gB = [self.comm.recv(g, self.cdtype, self.device) for _ in range(hi - lo)]
                gl = [self.comm.recv(g, self.rdtype, self.device) for _ in range((hi - lo) + (1 if g == 0 else 0))]
            for x, t in enumerate(gB):
                out_B[lo + x] = t
            first_bond = -1 if g == 0 else lo
            for x, t in enumerate(gl):
                out_l[first_bond + x + 1] = t
        return out_B, out_l
