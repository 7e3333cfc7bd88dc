"""Model check of the ticket schedule of the one-launch step (norm-first order
and the known-sync pass), on CPU.

compute-sanitizer is closed on the GPU pool and ncu cannot see a multi-rank
kernel, so the cross-rank protocol of ``nf_body`` (paper_2307_07950_b200/
csrc/selsync_step.cu) is also checked as a discrete-event model: N ranks of
G co-resident blocks; tickets in groups of N update tiles + 1 mean ticket;
tile t belongs to rank t % N; a rank's update of tile t is announced to the
owner's counter; a mean ticket of group g serves tile (g - lag) * N + rank
and waits for the agreed vote (unless the decision is known ahead) and for
all N announcements; a block claims its NEXT ticket before working on the
current one (the kernel's prefetch). Random block speeds, skewed rank start
times and the kernel's lag (grid / (N + 1) + 2, and smaller ones). Checked:
every ticket completes (no deadlock), a mean never starts before its tile's
N updates, every owned tile is averaged exactly once on sync steps, the
known-sync vote is posted only after the rank's last update tile.
"""

import heapq
import random

import pytest


def simulate(N, G, T, lag, known, sync, seed, norm_time=5.0):
    rng = random.Random(seed)
    groups = (T + N - 1) // N + lag
    total = groups * (N + 1)
    next_ticket = [0] * N
    cnt = [[0] * T for _ in range(N)]          # cnt[owner][tile]
    upd_done = [[False] * T for _ in range(N)]  # upd_done[rank][tile]
    updated_tiles = [0] * N
    averaged = [[0] * T for _ in range(N)]
    vote_post = [None] * N                      # time each rank posted its vote
    start = [rng.uniform(0.0, 3.0) for _ in range(N)]  # rank skew
    speed = [[rng.uniform(0.5, 2.0) for _ in range(G)] for _ in range(N)]
    events = []  # (time, seq, rank, block, ticket, is_poll)
    n_real = 0   # events that are not re-polls of a waiting block
    announce = []  # (time, rank, tile): update tile done + announced to the owner
    seq = 0

    def claim(r):
        k = next_ticket[r]
        next_ticket[r] += 1
        return k

    def ready(r, k, now):
        grp, pos = divmod(k, N + 1)
        if pos < N or k >= total:
            return True  # update tickets never wait
        m = grp - lag
        t = m * N + r
        if m < 0 or t >= T:
            return True
        vote_in = known or all(v is not None and v <= now for v in vote_post)
        return vote_in and (not sync or cnt[r][t] >= N)

    held = {}  # (rank, block) -> prefetched next ticket
    for r in range(N):
        if not known:
            vote_post[r] = start[r] + norm_time * rng.uniform(0.9, 1.1)  # norm sweep, then the vote
        t0 = start[r] + (0.0 if known else norm_time)
        for b in range(G):
            k = claim(r)
            held[r, b] = claim(r)  # the kernel prefetches the next ticket
            heapq.heappush(events, (t0, seq, r, b, k, False))
            n_real += 1
            seq += 1
    waiting = []
    finished = 0
    now = 0.0
    steps = 0
    while events or waiting:
        steps += 1
        assert steps < 10_000_000, "simulation does not terminate"
        vote_pending = [v for v in vote_post if v is not None and v > now]
        pollers = [(e[2], e[4]) for e in events if e[5]] + [(w[0], w[2]) for w in waiting]
        if (n_real == 0 and not announce and not vote_pending and pollers
                and not any(ready(pr, pk, now) for pr, pk in pollers)):
            # no block is working, no update and no vote is in flight: the waiters wait forever
            raise AssertionError(f"deadlock: {len(waiting) + len(events)} blocks waiting, none running")
        if not events:
            heapq.heappush(events, (min([a[0] for a in announce[:1]] + vote_pending), seq, -1, -1, -1, False))
            n_real += 1
            seq += 1
            continue
        now, _, r, b, k, is_poll = heapq.heappop(events)
        if not is_poll:
            n_real -= 1
        while announce and announce[0][0] <= now:
            _, ar, at = heapq.heappop(announce)
            upd_done[ar][at] = True
            cnt[at % N][at] += 1
            updated_tiles[ar] += 1
            if known and updated_tiles[ar] == T:
                vote_post[ar] = now  # the block finishing the rank's last tile posts the vote
        if r < 0:
            pass  # clock tick that delivered announcements
        elif k >= total:
            finished += 1
            # a block that runs past the last ticket is done; retry the waiters
        else:
            grp, pos = divmod(k, N + 1)
            if not ready(r, k, now):
                waiting.append((r, b, k))
            else:
                dur = 0.0
                if pos < N:
                    t = grp * N + pos
                    if t < T:
                        dur = speed[r][b]
                        # the tile's stores and its announcement land when the tile is done
                        heapq.heappush(announce, (now + dur, r, t))
                else:
                    m = grp - lag
                    t = m * N + r
                    if m >= 0 and t < T and sync:
                        assert all(upd_done[q][t] for q in range(N)), f"mean of tile {t} before all updates"
                        averaged[r][t] += 1
                        dur = 2.0 * speed[r][b]
                nxt = held[r, b]
                held[r, b] = claim(r)
                heapq.heappush(events, (now + dur, seq, r, b, nxt, False))
                n_real += 1
                seq += 1
        # wake every waiter at the current time (they re-check their condition)
        if waiting:
            for (wr, wb, wk) in waiting:
                heapq.heappush(events, (now + 0.01, seq, wr, wb, wk, True))
                seq += 1
            waiting = []
        if finished == N * G:
            break
    assert finished == N * G
    for r in range(N):
        assert updated_tiles[r] == T
        for t in range(T):
            want = 1 if (sync and t % N == r) else 0
            assert averaged[r][t] == want, (r, t, averaged[r][t])
        if known:
            assert vote_post[r] is not None
    return now


@pytest.mark.parametrize("N", [2, 4, 8])
@pytest.mark.parametrize("known,sync", [(False, True), (False, False), (True, True)],
                         ids=["norm-first-sync", "norm-first-local", "known-sync"])
def test_ticket_schedule_completes_and_orders_means(N, known, sync):
    G = 24
    for seed in range(6):
        T = random.Random(seed).choice([1, N - 1 if N > 1 else 1, 37, 101])
        base = G // (N + 1) + 2
        # the kernel's per-pass lags (nf_body): the known pass x3/4 over P2P,
        # the pass after the ||g||^2 sweep x3/2, and the base; plus the extremes
        scaled = (base - 2) * 3 // 4 + 2 if known else (base - 2) * 3 // 2 + 2
        for lag in sorted({base, scaled, 1, 0}):
            simulate(N, G, T, lag, known, sync, seed)


def test_model_detects_a_bad_schedule():
    """Teeth: a mean scheduled one group BEFORE its tile's updates (lag = -1)
    must deadlock with few blocks, and the model must say so."""
    with pytest.raises(AssertionError, match="deadlock|before all updates"):
        simulate(N=2, G=2, T=8, lag=-1, known=False, sync=True, seed=0)
