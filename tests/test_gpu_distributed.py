"""GPU checks of the multi-GPU frame pieces through the C
ABI, on the one B200 the test box has:

* nirc_collect_range shards concatenated in rank order == nirc_collect over
  all paths, row for row, bit for bit;
* nirc_train_grad over tile shards, summed, + nirc_train_apply ==
  nirc_train_step (the un-sharded fused step) within fp32 re-association;
* the whole sharded frame (distributed.run_frame_sharded) with two ranks
  sharing cuda:0 over a gloo group (NCCL refuses two ranks on one GPU):
  the row bands compose the 1-GPU image bit for bit, the training matches
  the 1-GPU frame, and the two cache replicas are bit-identical.
"""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2412_04634_b200 import _lib

    return _lib.load()


def _cornell(res=64):
    from paper_2412_04634_b200.scene import load_builtin

    return load_builtin("cornell").with_resolution(res, res)


def test_collect_range_shards_compose(lib):
    from paper_2412_04634_b200 import distributed as D
    from paper_2412_04634_b200.records import collect_training_records

    sc = _cornell(64)
    full = collect_training_records(sc, 3, 301, "nirc", frame=4)
    ops = D.DeviceOps()
    parts = []
    for r in range(3):
        p0, p1 = D.split_range(301, 3, r)
        parts.append(ops.collect_range(sc, 3, 4, p0, p1 - p0, "nirc"))
    got = torch.cat(parts, 0)
    want = D.pack_records({k: getattr(full, k) for k, _ in D.REC_COLS})
    assert got.shape == want.shape
    assert torch.equal(got, want)


@pytest.mark.parametrize("n", [700, 20000])
def test_train_grad_shards_match_train_step(lib, n):
    import nirc_oracle as O
    from paper_2412_04634_b200 import distributed as D
    from paper_2412_04634_b200.adam import AdamState
    from paper_2412_04634_b200.caches import Records, train_frame_device
    from paper_2412_04634_b200.mlp import init_theta, make_spec

    spec = make_spec(depth=4, table=2 ** 14)
    th0 = init_theta(spec, seed=5, out_scale=0.05)
    rec = Records(kind="nirc", frame=0, **O.synth_records(n, seed=8))
    # reference: the un-sharded fused step
    ta = torch.from_numpy(th0.copy()).cuda()
    res = train_frame_device(spec, ta, rec, seed=2, frame=1, steps=3)

    class C:  # the attributes DeviceOps reads from a Cache
        pass

    c = C()
    c.spec, c.theta, c.seed, c.frame = spec, torch.from_numpy(th0.copy()).cuda(), 2, 1
    c.loss_kind, c.loss_eps, c.adam = "relative_l2", 0.01, AdamState(th0)
    ops = D.DeviceOps()
    ntiles = ops.train_tiles(n, 16384)
    flags = torch.zeros((1,), dtype=torch.int32, device="cuda")
    trace = []
    for s in range(3):
        gsum = torch.zeros_like(c.theta)
        asum = torch.zeros((2,), dtype=torch.float64, device="cuda")
        for r in range(3):  # three "ranks" on one GPU
            g = torch.empty_like(c.theta)
            a = torch.zeros((2,), dtype=torch.float64, device="cuda")
            t0, t1 = D.split_range(ntiles, 3, r)
            ops.train_grad(c, rec, s, 16384, t0, t1, g, a, flags)
            gsum += g
            asum += a
        lo = torch.zeros((1,), dtype=torch.float64, device="cuda")
        ops.train_apply(c, gsum, asum, min(n, 16384), lo, flags)
        trace.append(float(lo.item()))
    assert int(flags.item()) == 0
    np.testing.assert_allclose(trace, res.trace, rtol=1e-6)
    assert c.adam.t == 3
    # hash-grid atomics and the shard sums re-associate fp32 additions; Adam
    # maps a ~1e-7 gradient change on a near-zero gradient to up to ~lr/1000.
    # A wrong shard moves parameters by ~lr = 1e-2.
    d = np.abs(c.theta.cpu().numpy() - ta.cpu().numpy())
    # a missing or doubled tile would move ~all touched parameters by ~lr
    assert (d > 1e-5).mean() < 1e-3 and d.max() < 5e-3 and d.mean() < 1e-7, (
        d.max(), d.mean(), (d > 1e-5).mean())


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _frame_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2412_04634_b200 import distributed as D
        from paper_2412_04634_b200.caches import Cache
        from paper_2412_04634_b200.frame import config3

        comm = D.Comm()
        sc = _cornell(96)
        cache = Cache.create("nirc", sc, seed=0, init="random")
        out = []
        for f in range(2):
            (img, img2, term), rows, st = D.run_frame_sharded(sc, cache, config3((8,)), comm,
                                                              seed=0, frame=f)
            full = D.gather_image(img, rows, comm)
            fterm = D.gather_image(term, rows, comm)
            out.append((full.cpu().numpy(), fterm.cpu().numpy(), st["trace"]))
        same = D.replicas_identical(cache, comm)
        q.put((rank, (out, cache.theta.cpu().numpy(), same)))
    except Exception:  # noqa: BLE001
        import traceback

        q.put((rank, "ERROR " + traceback.format_exc()))
    finally:
        import torch.distributed as dist

        if dist.is_initialized():
            dist.destroy_process_group()


def test_sharded_frame_two_ranks_one_gpu(lib):
    import torch.multiprocessing as mp

    from paper_2412_04634_b200.caches import Cache
    from paper_2412_04634_b200.frame import config3, run_frame

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_frame_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
    for v in res.values():
        assert not isinstance(v, str), v
    # the same two frames on one GPU
    sc = _cornell(96)
    cache = Cache.create("nirc", sc, seed=0, init="random")
    ref = []
    for f in range(2):
        (img, img2, term), st = run_frame(sc, cache, config3((8,)), seed=0, frame=f)
        ref.append((img.cpu().numpy(), term.cpu().numpy(), st.loss))
    for r in (0, 1):
        out, theta, same = res[r]
        assert same
        # frame 0 renders with the identical initial cache: bit-identical
        assert np.array_equal(out[0][0], ref[0][0])
        assert np.array_equal(out[0][1], ref[0][1])
        # frame 1 renders with the trained cache: same paths, close pixels
        assert np.array_equal(out[1][1], ref[1][1])
        np.testing.assert_allclose(out[1][0], ref[1][0], rtol=1e-3, atol=1e-4)
        np.testing.assert_allclose(out[1][2][-1], ref[1][2], rtol=1e-4)
        d = np.abs(theta - cache.theta.cpu().numpy())
        assert (d > 1e-5).mean() < 1e-2 and d.max() < 1e-2 and d.mean() < 1e-6, (
            d.max(), d.mean(), (d > 1e-5).mean())
    assert np.array_equal(res[0][1], res[1][1])


def _pipeline_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2412_04634_b200 import distributed as D
        from paper_2412_04634_b200.caches import Cache
        from paper_2412_04634_b200.frame import config3

        comm = D.Comm()
        sc = _cornell(96)
        outs = {}
        for mode in ("sequential", "overlapped"):
            cache = Cache.create("nirc", sc, seed=0, init="random")
            pipe = D.ShardedFramePipeline(sc, cache, config3((8,)), comm, seed=0)
            frames = []
            for f in range(3):
                if mode == "sequential":
                    (img, _, term), rows, st = D.run_frame_sharded(sc, cache, config3((8,)),
                                                                   comm, seed=0, frame=f)
                else:
                    (img, _, term), rows, st = pipe.step(f)
                    torch.cuda.current_stream().wait_stream(pipe.s_train)
                torch.cuda.synchronize()
                frames.append((D.gather_image(img, rows, comm).cpu().numpy(),
                               D.gather_image(term, rows, comm).cpu().numpy(),
                               st.get("records"), st.get("trace")))
            outs[mode] = (frames, cache.theta.cpu().numpy(), D.replicas_identical(cache, comm))
        q.put((rank, outs))
    except Exception:  # noqa: BLE001
        import traceback

        q.put((rank, "ERROR " + traceback.format_exc()))
    finally:
        import torch.distributed as dist

        if dist.is_initialized():
            dist.destroy_process_group()


def test_overlapped_sharded_frames_match_sequential(lib):
    """ShardedFramePipeline (render(f) || all-gather + sharded train(f) on a
    second stream, frame f+1's records walked in frame f's launch) against
    run_frame_sharded on two ranks sharing one GPU: the same frames -- path
    lengths, record counts, loss traces, images and the final theta (the
    deterministic scatter makes the sums order-free) -- and identical
    replicas."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pipeline_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=900) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
    for v in res.values():
        assert not isinstance(v, str), v
    for r in (0, 1):
        seq, ovl = res[r]["sequential"], res[r]["overlapped"]
        assert seq[2] and ovl[2]
        for (i0, t0, n0, tr0), (i1, t1, n1, tr1) in zip(seq[0], ovl[0]):
            assert np.array_equal(t0, t1)
            assert n0 == n1
            np.testing.assert_allclose(tr1, tr0, rtol=1e-6)
            np.testing.assert_allclose(i1, i0, rtol=1e-6, atol=1e-9)
        np.testing.assert_allclose(ovl[1], seq[1], rtol=1e-6, atol=1e-9)
    np.testing.assert_array_equal(res[0]["overlapped"][1], res[1]["overlapped"][1])
