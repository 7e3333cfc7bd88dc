"""World-size-2 tests of the rank-group logic over gloo on CPU (no GPU).

Covers what the NCCL path does across B200s -- C1 agreement (allreduce-MAX ==
OR of votes, errors reaching every rank), C2 averaging, bootstrap broadcast --
and drives a 2-rank SelSync protocol through those collectives with the
package's native scalar signal API, checked bit-for-bit against the oracle's
N=2 restatement of _selsync_step + the parameter server."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import selsync_oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2307_07950_b200 import DeltaThreshold, GradSignalState, decide, observe, relative_change
        from paper_2307_07950_b200.collectives import RankGroup

        g = RankGroup()
        assert (g.size, g.rank) == (world, rank)
        res = {}
        # C1: MAX of 0/1 words is the OR of the votes
        for votes in ([0, 0], [1, 0], [0, 1], [1, 1]):
            w = torch.tensor([votes[rank]], dtype=torch.int32)
            g.agree(w)
            res[f"agree_{votes}"] = int(w)
        # an error word (>= 2) on one rank reaches every rank
        w = torch.tensor([2 if rank == 1 else 1], dtype=torch.int32)
        g.agree(w)
        res["err"] = int(w)
        # C2 average / sum / bootstrap broadcast
        v = torch.arange(4, dtype=torch.float64) + 10 * rank
        g.average_(v)
        res["avg"] = v.numpy().copy()
        v = torch.full((3,), float(rank + 1))
        g.sum_(v)
        res["sum"] = v.numpy().copy()
        b = torch.full((5,), float(rank))
        g.broadcast_(b, 0)
        res["bcast"] = b.numpy().copy()

        # 2-rank SelSync protocol through the collectives (parameter aggregation)
        d, steps, seed, delta, warmup, lam, lr = 40, 40, 21, 0.2, 3, 0.5, 0.05
        P = 2 * d + 2
        params = torch.tensor(O.init_params_linear(d, 9) if rank == 0 else np.zeros(P))
        g.broadcast_(params, 0)  # replicas start identical
        st = GradSignalState(smoothing=lam, warmup=warmup)
        thr = DeltaThreshold(delta)
        trace = []
        for s in range(steps):
            grad = O.synthetic_grad32(seed, rank, s, P).astype(np.float64)
            st = observe(st, float(grad @ grad))
            dg = relative_change(st) if st.step_count >= 2 else float("nan")
            params = params - lr * torch.from_numpy(grad)  # local update lands first
            word = torch.tensor([1 if decide(st, thr) == "sync" else 0], dtype=torch.int32)
            g.agree(word)
            if int(word) == 1:
                g.average_(params)
            trace.append((st.ewma_current, dg, int(word)))
        res["trace"] = np.array(trace)
        res["params"] = params.numpy().copy()
        np.save(os.path.join(outdir, f"rank{rank}.npy"), res, allow_pickle=True)
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def results(tmp_path_factory):
    out = tmp_path_factory.mktemp("gloo")
    mp.spawn(_worker, args=(2, _free_port(), str(out)), nprocs=2, join=True)
    return [np.load(out / f"rank{r}.npy", allow_pickle=True).item() for r in range(2)]


def test_agree_is_or_of_votes(results):
    for r in results:
        assert r["agree_[0, 0]"] == 0
        assert r["agree_[1, 0]"] == r["agree_[0, 1]"] == r["agree_[1, 1]"] == 1
        assert r["err"] == 2


def test_average_sum_broadcast(results):
    for r in results:
        np.testing.assert_array_equal(r["avg"], np.arange(4) + 5.0)
        np.testing.assert_array_equal(r["sum"], [3.0, 3.0, 3.0])
        np.testing.assert_array_equal(r["bcast"], np.zeros(5))


def test_two_rank_protocol_matches_oracle(results):
    d, steps, seed, delta, warmup, lam, lr = 40, 40, 21, 0.2, 3, 0.5, 0.05
    P = 2 * d + 2
    ref = O.simulate_selsync(O.init_params_linear(d, 9), 2, steps,
                             lambda w, s, _p: O.synthetic_grad32(seed, w, s, P),
                             delta=delta, warmup=warmup, smoothing=lam, lr=lr)
    assert 0 < ref.decision.sum() < steps
    for rank, r in enumerate(results):
        np.testing.assert_array_equal(r["trace"][:, 0], ref.ewma[:, rank])
        np.testing.assert_array_equal(r["trace"][:, 1], ref.delta_g[:, rank])
        np.testing.assert_array_equal(r["trace"][:, 2].astype(bool), ref.decision)
        np.testing.assert_array_equal(r["params"], ref.finals[rank])
