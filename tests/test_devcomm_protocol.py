"""An executable model of the device-initiated comm protocol (kernels.h DevComm),
run by W threads -- one per rank -- with random delays between every step, so that the
ranks drift arbitrarily far apart within what the protocol allows.

It checks the protocol's claims that the GPU code relies on but one GPU cannot exercise:
  - the accumulator inbox slots [generation parity][pAp, rr][sender] are never overwritten
    before every rank has consumed them (each consumed sum must equal the sum of the values
    the ranks pushed for exactly that reduction),
  - the halo of p_(k+1), pushed straight into the receiver's p array, never overwrites the
    halo of p_k before the receiver's SpMV(k) has read it,
  - consecutive solves (generations) and solves that stop early (a uniform decision) reuse
    the regions safely,
  - with ONE generation parity instead of two, a fast rank starting the next solve CAN
    overwrite a slot a slow rank still has to read (the model finds it: the test has teeth).
The sequence numbers and slot indices are those of kernels.h (comm_seq, comm_halo_seq,
comm_acc_flag), written out here.
"""
import random
import threading
import time

import pytest

SEQ_SHIFT = 21          # kernels.h comm_seq: (gen << 21) + 2k + which; halo: (gen << 21) + k


def comm_seq(gen, k, which):
    return (gen << SEQ_SHIFT) + 2 * k + which


def comm_halo_seq(gen, k):
    return (gen << SEQ_SHIFT) + k


class Region:
    """One rank's comm region: acc flags / inbox [gen parity][which][sender], halo flags and
    the halo columns of its p array, [sender]."""

    def __init__(self, W, parities):
        self.P = parities
        self.acc_flag = [[[0] * W for _ in range(2)] for _ in range(parities)]
        self.inbox = [[[None] * W for _ in range(2)] for _ in range(parities)]
        self.halo_flag = [0] * W
        self.halo = [None] * W


class Failure(Exception):
    pass


def run_model(W, solves, parities=2, seed=0, max_delay=2e-4, timeout=20.0):
    rnd = random.Random(seed)
    regions = [Region(W, parities) for _ in range(W)]
    nbrs = [sorted({(r - 1) % W, (r + 1) % W} - {r}) for r in range(W)]
    errors = []
    lock = threading.Lock()
    delays = [[rnd.random() * max_delay for _ in range(4000)] for _ in range(W)]

    def val(r, gen, k, which):              # what rank r contributes to a reduction
        return (r + 1) * 1_000_003 + gen * 10_007 + k * 31 + which

    def run(r):
        d = iter(delays[r])

        def pause():
            time.sleep(next(d, 0.0))

        def spin(cond):
            t0 = time.time()
            while not cond():
                if time.time() - t0 > timeout:
                    raise Failure(f"rank {r}: timeout")
                time.sleep(0)

        def push_acc(gen, k, which, v):     # k_acc_push / acc_push_last_cta
            gp = gen % parities
            for t in range(W):
                regions[t].inbox[gp][which][r] = (gen, k, which, v)
            pause()
            for t in range(W):
                regions[t].acc_flag[gp][which][r] = comm_seq(gen, k, which)

        def consume(gen, k, which):          # acc_in_load: acquire W flags, sum W slots
            gp = gen % parities
            seq = comm_seq(gen, k, which)
            me = regions[r]
            spin(lambda: all(me.acc_flag[gp][which][t] >= seq for t in range(W)))
            pause()
            got = [me.inbox[gp][which][t] for t in range(W)]
            want = [(gen, k, which, val(t, gen, k, which)) for t in range(W)]
            if got != want:
                raise Failure(f"rank {r}: reduction (gen {gen}, k {k}, which {which}) read "
                              f"{got}, expected {want}")

        def push_halo(gen, k_halo):          # k_push: store into the receivers' p, then flag
            for q in nbrs[r]:
                regions[q].halo[r] = (gen, k_halo)
            pause()
            for q in nbrs[r]:
                regions[q].halo_flag[r] = comm_halo_seq(gen, k_halo)

        def wait_halo(gen, k):               # k_halo_wait / the tail of K7
            me = regions[r]
            spin(lambda: all(me.halo_flag[q] >= comm_halo_seq(gen, k) for q in nbrs[r]))

        def spmv_reads_halo(gen, k):         # SpMV(k) reads p_k's halo columns
            me = regions[r]
            for q in nbrs[r]:
                if me.halo[q] != (gen, k):
                    raise Failure(f"rank {r}: SpMV({k}) of gen {gen} saw halo {me.halo[q]} "
                                  f"from rank {q}")

        try:
            for gen, (K, stop_at) in enumerate(solves, start=1):
                pause()
                push_acc(gen, 0, 1, val(r, gen, 0, 1))          # init: rr_0
                consume(gen, 0, 1)
                push_halo(gen, 1)                               # halo of p_1 = b
                wait_halo(gen, 1)
                for k in range(1, K + 1):
                    pause()
                    spmv_reads_halo(gen, k)
                    pause()
                    push_acc(gen, k, 0, val(r, gen, k, 0))      # SpMV's last CTA: pAp_k
                    consume(gen, k, 0)                          # K6 prologue
                    push_acc(gen, k, 1, val(r, gen, k, 1))      # K6's last CTA: rr_k
                    last = k == K or k == stop_at
                    if not last:
                        push_halo(gen, k + 1)                   # k_push before K7
                    consume(gen, k, 1)                          # K7 prologue (stop decision)
                    if last:
                        break
                    wait_halo(gen, k + 1)                       # K7's last CTA
        except Failure as e:
            with lock:
                errors.append(str(e))

    threads = [threading.Thread(target=run, args=(r,)) for r in range(W)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    return errors


@pytest.mark.parametrize("W", [2, 3, 4])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_protocol_safe_under_random_schedules(W, seed):
    # three solves: run to the cap, stop early (uniformly) at k = 4, run to the cap again
    errs = run_model(W, [(12, None), (12, 4), (9, None)], seed=seed)
    assert not errs, errs[:3]


def test_one_generation_parity_is_not_enough():
    """With a single inbox parity a rank that races into the next solve overwrites rr_K's
    slot (its rr_0 lands in the same [which = rr] slot) before a slow rank has read it."""
    found = False
    for seed in range(40):
        # rank 0 fast, the others slow: delays chosen by the seed; one parity
        errs = run_model(3, [(3, None), (3, None), (3, None)], parities=1, seed=seed,
                         max_delay=2e-3, timeout=2.0)
        if errs:
            found = True
            break
    assert found, "the model should expose the single-parity race"
