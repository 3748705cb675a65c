"""CPU model of the flag-free small/mid-size protocols' scratch reuse.

The one-shot kernel (ar_ll_kernel) and the LL128 two-shot kernel (ar_ll128_kernel) carry no
entry or exit barrier: a rank writes its lines for call e into its peers' scratch slot of
parity e & 1 without asking whether the peer is done with that slot, and reads its own slots
until their flags equal e.  The claimed invariant: a slot of parity p is rewritten (call e)
only after its reader consumed the previous use (call e − 2), because the writer finished call
e − 1, which needed lines the reader wrote in ITS call e − 1, which it started only after
finishing call e − 2 (stream order).

This module executes that protocol under random schedules — every rank a sequence of calls,
each call a sequence of writes (always enabled) and flag-checked reads (enabled once the
awaited line carries the call's epoch) — and asserts that no write ever lands on a line whose
current content has not been read yet, and that every schedule completes.  A single-buffered
one-shot variant (parity removed) must violate the invariant: the model can fail.  (Each slot
stands for all lines one writer sends one reader in a call; the argument is per line.)"""
import random

import pytest


def run(world, calls, protocol, parities=2, seed=0):
    """Returns (violations, completed).  protocol: "ll" (every rank sends its whole input to
    every peer, reads all peers) or "ll128" (RS: send slice b to owner b; owner reads N − 1
    slices, then AG: owner sends its result to every peer, which reads N − 1 results)."""
    rnd = random.Random(seed)
    # scratch[area][reader][parity][writer] = (epoch written, consumed?)
    areas = 1 if protocol == "ll" else 2
    scratch = [[[[(0, True) for _ in range(world)] for _ in range(parities)] for _ in range(world)]
               for _ in range(areas)]
    violations = []

    def program(r, e):
        par = e % parities
        ops = []
        peers = [q for q in range(world) if q != r]
        if protocol == "ll":
            ops += [("w", 0, q, par, r) for q in peers]          # my lines into every peer
            ops += [("r", 0, r, par, q) for q in peers]          # every peer's lines into me
        else:
            ops += [("w", 0, q, par, r) for q in peers]          # RS: my slice of block q -> owner q
            ops += [("r", 0, r, par, q) for q in peers]          # reduce my block
            ops += [("w", 1, q, par, r) for q in peers]          # AG: my result -> every peer
            ops += [("r", 1, r, par, q) for q in peers]          # gather the others' results
        return ops

    state = [[r, 1, program(r, 1), 0] for r in range(world)]     # rank, epoch, ops, pc
    done = [False] * world
    steps = 0
    while not all(done):
        ready = []
        for r in range(world):
            if done[r]:
                continue
            _, e, ops, pc = state[r]
            kind, area, reader, par, writer = ops[pc]
            if kind == "w":
                ready.append(r)
            elif scratch[area][reader][par][writer][0] == e:
                ready.append(r)
        if not ready:
            return violations, False                               # deadlock
        r = rnd.choice(ready)
        _, e, ops, pc = state[r]
        kind, area, reader, par, writer = ops[pc]
        if kind == "w":
            old_e, consumed = scratch[area][reader][par][writer]
            if not consumed:
                violations.append((r, e, area, reader, par, writer, old_e))
            scratch[area][reader][par][writer] = (e, False)
        else:
            scratch[area][reader][par][writer] = (e, True)
        state[r][3] += 1
        if state[r][3] == len(ops):                                 # call complete (stream order)
            if e == calls:
                done[r] = True
            else:
                state[r] = [r, e + 1, program(r, e + 1), 0]
        steps += 1
    return violations, True


@pytest.mark.parametrize("protocol", ["ll", "ll128"])
@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_double_buffered_scratch_is_safe(protocol, world):
    for seed in range(40):
        violations, completed = run(world, 6, protocol, parities=2, seed=seed)
        assert completed, f"deadlock (seed {seed})"
        assert not violations, f"a line was overwritten before it was read: {violations[:3]} (seed {seed})"


def test_single_buffer_would_be_unsafe_for_the_one_shot_protocol():
    """Negative control: with one scratch buffer the one-shot protocol lets a fast rank
    overwrite lines a slow peer has not read yet — the model detects it (so the safety test
    above has teeth)."""
    found = False
    for seed in range(200):
        violations, _ = run(4, 6, "ll", parities=1, seed=seed)
        if violations:
            found = True
            break
    assert found


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_two_shot_protocol_is_safe_even_single_buffered(world):
    """The LL128 two-shot protocol is causally ordered: a rank's call e + 1 RS lines reach
    owner o only after this rank read o's call-e AG result, which o wrote after reading every
    call-e RS line; an owner's call e + 1 AG lines need every reader's call e + 1 RS lines,
    sent after the reader finished call e.  So even one buffer would be safe (the kernel keeps
    the parity planes anyway, like the one-shot kernel)."""
    for seed in range(40):
        violations, completed = run(world, 6, "ll128", parities=1, seed=seed)
        assert completed and not violations
