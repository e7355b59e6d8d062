"""The peer transport's ordering protocol (csrc/kmf_peer.cuh), model-checked
on the CPU: every rank is a state machine running exactly the device
sequence of one RK stage -- wait for the peers' pushes, read the halo (band
pass), publish "read", wait for the peers it pushes into, push (update),
publish the push, and at stage 4 the limb all-gather -- and a random
scheduler interleaves the ranks' steps.  Over many schedules and
topologies (ring = sectors, path = bands, random one-way links) the model
checks what the GPU counters must guarantee: no deadlock; a rank never
overwrites a peer's halo while that peer is reading it; every halo read
sees exactly the version of the stage being computed; no limb row is
overwritten before every rank has summed it.  (The hardware tests run the
real kernels on one GPU; this covers the interleavings a single device
does not produce.)"""

from __future__ import annotations

import random

import pytest


class Rank:
    def __init__(self, r, recv, send, nranks):
        self.r, self.recv, self.send, self.n = r, recv, send, nranks
        # device counters (PeerFlags): what peers published here
        self.data = [0] * nranks
        self.read = [0] * nranks
        self.limb_seq = [0] * nranks
        self.gather = [[None] * nranks for _ in range(2)]
        # own counters
        self.pushes = self.bands = self.iters = 0
        self.summed = 0  # model only: last iteration whose limb rows this rank summed
        # halo contents: version of q each sender last pushed here
        self.halo = {p: 0 for p in recv}
        self.reading = False
        self.pc = 0
        self.stage = 0


def program(rank, stages):
    """The per-stage device sequence of kmf_b200.cu enqueue_tail (peer
    branch) as a list of steps; each step returns False while blocked."""
    steps = []
    for t in range(1, stages + 1):
        steps += [("wait_data", t), ("read_begin", t), ("band_done", t), ("wait_read", t), ("push", t),
                  ("pushed", t)]
        if t % 4 == 0:
            steps += [("limbs_write", t), ("limbs_wait", t), ("limbs_sum", t)]
    steps.append(("wait_data_end", stages))
    return steps


def step(ranks, rk, op, t, log):
    me = ranks[rk]
    if op in ("wait_data", "wait_data_end", "wait_read", "limbs_wait"):
        return True  # readiness: step_ready (the spin loops of kmf_peer.cuh)
    if op == "read_begin":
        for p in me.recv:  # the halo must hold the version of this stage's q
            assert me.halo[p] == me.pushes, (rk, p, me.halo[p], me.pushes, t)
        me.reading = True
        return True
    if op == "band_done":
        me.reading = False
        me.bands += 1
        for p in me.recv:
            ranks[p].read[rk] = me.bands
        return True
    if op == "push":
        for p in me.send:
            assert not ranks[p].reading, f"rank {rk} overwrote rank {p}'s halo during its band pass (stage {t})"
            ranks[p].halo[rk] = me.pushes + 1
        return True
    if op == "pushed":
        me.pushes += 1
        for p in me.send:
            ranks[p].data[rk] = me.pushes
        return True
    if op == "limbs_write":
        it = me.iters + 1
        for p in range(me.n):
            if p != rk:
                row = ranks[p].gather[it & 1]
                # the row of parity it&1 from me must have been summed by p
                # (p's iteration it-2 sum) before I overwrite it
                assert row[rk] is None or ranks[p].summed >= row[rk], (rk, p, it, row[rk], ranks[p].summed)
                row[rk] = it
        me.iters = it
        for p in range(me.n):
            if p != rk:
                ranks[p].limb_seq[rk] = it
        return True
    if op == "limbs_sum":
        for p in range(me.n):
            if p != rk:
                assert me.gather[me.iters & 1][p] == me.iters, (rk, p, me.gather[me.iters & 1][p], me.iters)
        me.summed = me.iters
        return True
    raise AssertionError(op)


def run(topology, stages, seed, bias=0.0):
    """bias: probability of stepping the lowest-numbered ready rank (starves
    the high ranks -- the adversarial schedules uniform picks rarely make)."""
    n = len(topology)
    send = {r: sorted(topology[r]) for r in range(n)}
    recv = {r: sorted(p for p in range(n) if r in topology[p]) for r in range(n)}
    ranks = [Rank(r, recv[r], send[r], n) for r in range(n)]
    progs = [program(r, stages) for r in range(n)]
    rng = random.Random(seed)
    log = []
    while True:
        live = [r for r in range(n) if ranks[r].pc < len(progs[r])]
        if not live:
            return ranks
        ready = [r for r in live if step_ready(ranks, r, progs[r][ranks[r].pc])]
        assert ready, f"deadlock: pcs {[ranks[r].pc for r in range(n)]}"
        r = ready[0] if rng.random() < bias else rng.choice(ready)
        op, t = progs[r][ranks[r].pc]
        assert step(ranks, r, op, t, log)
        ranks[r].pc += 1


def step_ready(ranks, rk, instr):
    op, _ = instr
    me = ranks[rk]
    if op in ("wait_data", "wait_data_end"):
        return all(me.data[p] >= me.pushes for p in me.recv)
    if op == "wait_read":
        return all(me.read[p] >= me.bands for p in me.send)
    if op == "limbs_wait":
        return all(me.limb_seq[p] >= me.iters for p in range(me.n) if p != rk)
    return True


def ring(n):
    return [{(r - 1) % n, (r + 1) % n} - {r} for r in range(n)]


def path(n):
    return [{p for p in (r - 1, r + 1) if 0 <= p < n} for r in range(n)]


@pytest.mark.parametrize("n", [2, 3, 4, 8, 16])
@pytest.mark.parametrize("shape", ["ring", "path"])
def test_protocol_random_schedules(n, shape):
    topo = ring(n) if shape == "ring" else path(n)
    for seed in range(60):
        for bias in (0.0, 0.9, 0.99):
            ranks = run(topo, stages=12, seed=seed, bias=bias)
            assert all(r.pushes == 12 and r.bands == 12 and r.iters == 3 for r in ranks)


def test_protocol_one_way_links():
    """Stencils need not be symmetric: rank r may receive from p without
    sending to it (kNN neighbourhoods) -- the masks are per direction."""
    rng = random.Random(5)
    for trial in range(40):
        n = rng.randint(2, 6)
        topo = [set() for _ in range(n)]
        for r in range(n):
            for p in range(n):
                if p != r and rng.random() < 0.45:
                    topo[r].add(p)
        run(topo, stages=8, seed=trial, bias=0.9 if trial % 2 else 0.0)


@pytest.mark.parametrize("drop", ["wait_read", "limbs_parity"])
def test_model_catches_a_broken_protocol(drop):
    """Sanity of the model itself: without the read wait before the push
    (the WAR guard) some schedule overwrites a halo mid-read; with a single
    limb row instead of one per iteration parity, some schedule overwrites
    a row before a slow rank summed it -- on 16 ranks in bands: an
    iteration's four stages chain the ranks 8 hops apart (band waits on the
    neighbours' previous update, update on their band pass), so up to ~9
    ranks the halo waits alone would keep a single row safe."""
    global step_ready
    keep, keep_step = step_ready, globals()["step"]

    def no_read_wait(ranks, rk, instr):
        return True if instr[0] == "wait_read" else keep(ranks, rk, instr)

    def one_row(ranks, rk, op, t, log):
        if op in ("limbs_write", "limbs_sum"):  # parity 0 only: a single row
            for r in ranks:
                r.gather[1] = r.gather[0]
        return keep_step(ranks, rk, op, t, log)

    if drop == "wait_read":
        step_ready = no_read_wait
    else:
        globals()["step"] = one_row
    try:
        with pytest.raises(AssertionError, match="overwrote|\\("):
            for seed in range(400):
                run(ring(4) if drop == "wait_read" else path(16), stages=16, seed=seed, bias=0.99)
    finally:
        step_ready = keep
        globals()["step"] = keep_step
