"""Host logic of the multi-GPU frame (paper_2412_04634_b200/distributed.py)
on CPU: world_size-2 gloo process groups, with the per-rank compute supplied
by a checker built on the oracle (the B200 box has one GPU per process; the
same code drives the C ABI there).  Pins:

* shard arithmetic (contiguous, disjoint, balanced, covering);
* variable-length record all-gather in rank order == the 1-GPU row order;
* sharded training (tile shards + all-reduced gradient + identical Adam)
  matches the un-sharded oracle step and leaves bit-identical replicas;
* error semantics (bad pdf seen by ONE rank raises on every rank).
"""

import os
import socket
import types

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import nirc_oracle as O
from paper_2412_04634_b200 import distributed as D

TILE = 128  # rows per fused training tile (train_fused.cu kTR)


def test_split_range_partitions():
    for n in (0, 1, 5, 64, 1080, 2160, 51840, 257):
        for world in (1, 2, 3, 4, 8):
            spans = [D.split_range(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        D.split_range(10, 2, 2)


def test_pack_unpack_roundtrip():
    rec = O.synth_records(37, seed=2)
    cols = {k: torch.from_numpy(np.ascontiguousarray(v)) for k, v in rec.items()}
    packed = D.pack_records(cols)
    assert packed.shape == (37, D.REC_WIDTH)
    back = D.unpack_records(packed, "nirc", 3)
    for k, v in rec.items():
        assert np.array_equal(back.__dict__[k].numpy(), v), k
    assert back.frame == 3 and len(back) == 37


# ------------------------------------------------------------ oracle ops --
class FakeAdam:
    def __init__(self, n):
        self.o = O.Adam(n)
        self.m = torch.from_numpy(self.o.m)
        self.v = torch.from_numpy(self.o.v)
        self._t = torch.zeros((1,), dtype=torch.int64)
        self._skipped = torch.zeros((1,), dtype=torch.int64)
        self.lr = self.o.lr


def fake_cache(spec, seed, frame=0, loss="relative_l2"):
    theta = torch.from_numpy(O.init_theta(spec, seed=seed, out_scale=0.05))
    return types.SimpleNamespace(spec=spec, theta=theta, adam=FakeAdam(spec.theta_len),
                                 seed=seed, frame=frame, loss_kind=loss, loss_eps=0.01,
                                 record_kind="nirc", scene=None)


def fake_path_records(p):
    """Deterministic stand-in for walk_record: path p yields p % 3 rows."""
    rows = []
    for k in range(p % 3):
        r = O.synth_records(1, seed=1000 + 7 * p + k)
        rows.append(np.concatenate([r[c].reshape(1, w) for c, w in D.REC_COLS], axis=1))
    return np.concatenate(rows, axis=0) if rows else np.zeros((0, D.REC_WIDTH))


class OracleOps:
    """Per-rank compute restated with the oracle (the checker)."""

    def collect_range(self, scene, seed, frame, path0, count, kind):
        rows = [fake_path_records(p) for p in range(path0, path0 + count)]
        return torch.from_numpy(np.concatenate(rows, axis=0) if rows
                                else np.zeros((0, D.REC_WIDTH)))

    def train_tiles(self, n, cap):
        return (min(n, cap) + TILE - 1) // TILE

    def train_grad(self, cache, records, step, cap, t0, t1, grad, aux, flags):
        spec, theta = cache.spec, cache.theta.numpy()
        rec = {k: getattr(records, k).numpy() for k, _ in D.REC_COLS}
        n = len(records)
        idx = O.select_batch(cache.seed, cache.frame, step, n, cap)
        B = idx.shape[0]
        rows = idx[t0 * TILE: min(t1 * TILE, B)]
        g = np.zeros_like(theta)
        lsum = 0.0
        bad = 0.0
        if rows.size:
            X, ent, wts = O.encode_batch(spec, theta, rec["pos"][rows], rec["ns"][rows],
                                         rec["alb"][rows], rec["rough"][rows], rec["dirs"][rows])
            y, c = O.mlp_forward(spec, theta, X, training=True)
            t, pdf = rec["target"][rows], rec["pdf"][rows]
            bad = float(np.any(pdf <= 0.0))
            den = y * y + np.float32(cache.loss_eps)
            p = pdf[:, None]
            diff = y - t
            lsum = float((diff * diff / (p * den)).sum())
            dy = (2.0 * diff / (p * den) / (B * 3)).astype(np.float32)
            g = O.mlp_backward(spec, theta, c, dy, ent, wts)
        grad.copy_(torch.from_numpy(g))
        aux[0] = lsum
        aux[1] = bad

    def train_apply(self, cache, grad, aux, batch, loss_out, flags):
        if int(flags[0]) & 3:
            return
        if float(aux[1]) > 0:
            flags[0] |= 1
            return
        loss = float(aux[0]) / (batch * 3)
        loss_out[0] = loss
        if not np.isfinite(loss):
            flags[0] |= 2
            return
        th = cache.theta.numpy()
        if cache.adam.o.step(th, grad.numpy()):
            cache.adam._t[0] += 1
        else:
            cache.adam._skipped[0] += 1


# --------------------------------------------------------------- workers --
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(world, fn, *args):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, fn, args)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r, res = q.get(timeout=300)
        out[r] = res
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    errs = [v for v in out.values() if isinstance(v, str) and v.startswith("ERROR")]
    assert not errs, errs[0]
    return out


def _worker(rank, world, port, q, fn, args):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        q.put((rank, fn(D.Comm(), *args)))
    except Exception as e:  # noqa: BLE001 -- reported to the parent
        import traceback

        q.put((rank, "ERROR " + traceback.format_exc() + repr(e)))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def _gather_job(comm, n_local):
    t = torch.arange(n_local[comm.rank] * 2, dtype=torch.float64).reshape(-1, 2) + 100 * comm.rank
    return comm.all_gather_rows(t).numpy()


def test_all_gather_rows_rank_order():
    n_local = [3, 0]
    out = _run(2, _gather_job, n_local)
    want = np.concatenate([np.arange(6.0).reshape(3, 2), np.zeros((0, 2))])
    assert np.array_equal(out[0], want) and np.array_equal(out[1], want)


def _collect_job(comm, count):
    cache = fake_cache(O.Spec(table=2 ** 10, depth=2), seed=4)
    rec = D.collect_sharded(cache, comm, count=count, frame=5, ops=OracleOps())
    return D.pack_records({k: getattr(rec, k) for k, _ in D.REC_COLS}).numpy()


def test_collect_sharded_matches_path_order():
    count = 41
    out = _run(2, _collect_job, count)
    want = np.concatenate([fake_path_records(p) for p in range(count)])
    assert np.array_equal(out[0], want)
    assert np.array_equal(out[1], want)


def _train_job(comm, n, steps, cap):
    spec = O.Spec(table=2 ** 10, depth=2)
    cache = fake_cache(spec, seed=9, frame=2)
    rec = D.unpack_records(torch.from_numpy(np.concatenate(
        [O.synth_records(n, seed=11)[k].reshape(n, w) for k, w in D.REC_COLS], axis=1)),
        "nirc", 2)
    trace = D.train_frame_sharded(cache, rec, comm, steps=steps, batch=cap, ops=OracleOps())
    same = D.replicas_identical(cache, comm)
    return trace, cache.theta.numpy().copy(), cache.frame, same, int(cache.adam._t[0])


@pytest.mark.parametrize("n,cap", [(300, 16384), (1000, 256)])
def test_sharded_training_matches_single_gpu(n, cap):
    steps = 3
    out = _run(2, _train_job, n, steps, cap)
    # un-sharded oracle steps (caches.py:310-354)
    spec = O.Spec(table=2 ** 10, depth=2)
    theta = O.init_theta(spec, seed=9, out_scale=0.05)
    adam = O.Adam(spec.theta_len)
    rec = O.synth_records(n, seed=11)
    ref = []
    for s in range(steps):
        v, _ = O.train_step(spec, theta, adam, rec, seed=9, frame=2, step=s, cap=cap)
        ref.append(v)
    for r in (0, 1):
        trace, th, frame, same, t = out[r]
        assert same, "replicas diverged"
        assert frame == 3 and t == steps
        np.testing.assert_allclose(trace, ref, rtol=1e-6)
        # Adam turns fp32 re-association of the gradient sum (~1e-7 rel) into
        # ~1e-5 relative parameter differences; a wrong shard would be off by lr
        np.testing.assert_allclose(th, theta, rtol=1e-4, atol=2e-6)
    assert np.array_equal(out[0][1], out[1][1])


def _bad_pdf_job(comm):
    spec = O.Spec(table=2 ** 10, depth=2)
    cache = fake_cache(spec, seed=9)
    n = 200
    r = O.synth_records(n, seed=11)
    idx = O.select_batch(9, 0, 0, n, 16384)
    r["pdf"][idx[-1]] = 0.0  # a row of the LAST tile: only rank 1 sees it
    rec = D.unpack_records(torch.from_numpy(np.concatenate(
        [r[k].reshape(n, w) for k, w in D.REC_COLS], axis=1)), "nirc", 0)
    from paper_2412_04634_b200.errors import InvalidSampleError

    try:
        D.train_frame_sharded(cache, rec, comm, steps=2, ops=OracleOps())
    except InvalidSampleError:
        return "raised", cache.frame, int(cache.adam._t[0])
    return "no-raise", cache.frame, int(cache.adam._t[0])


def test_bad_pdf_on_one_rank_raises_everywhere():
    out = _run(2, _bad_pdf_job)
    assert out[0] == out[1] == ("raised", 0, 0)
