"""Tensor-parallel PPMoE over real NCCL (one process per GPU) vs the single-process
simulated world: same outputs and gradients (the reference's T-rank semantics,
moe.py:254-313).  Needs >= 2 GPUs; skipped otherwise."""

import os
import queue as _queue
import time

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _collect(q, procs, timeout=240):
    """Results from the worker processes; fail fast if one of them dies."""
    got, t0 = {}, time.time()
    while len(got) < len(procs):
        try:
            r, res = q.get(timeout=2)
            got[r] = res
        except _queue.Empty:
            dead = [p.exitcode for p in procs if p.exitcode not in (None, 0)]
            if dead:
                for p in procs:
                    p.kill()
                raise AssertionError(f"worker process failed with exit code {dead}")
            if time.time() - t0 > timeout:
                for p in procs:
                    p.kill()
                raise AssertionError("timed out waiting for the worker processes")
    return got


def _test_override(n, k, e):
    """A fixed routing with k distinct experts per token (route_override, moe.py:273-285)."""
    g = torch.Generator().manual_seed(123)
    return torch.stack([torch.randperm(e, generator=g)[:k] for _ in range(n)]).to("cuda")


def _worker(rank, world, port, q, k, cf, env=None, e=8):
    import torch.distributed as dist

    os.environ.update(env or {})

    import paper_2304_11414_b200 as P

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        h, n = 512, int(os.environ.get("_TEST_N", "1024"))
        el = e // world
        full = P.MoeLayerWeights.random(h, e, seed=11, device="cuda")  # identical on every rank
        local = P.MoeLayerWeights(P.GateParams(full.gate.wg.detach().clone().requires_grad_()),
                                  full.bank.slice(rank * el, (rank + 1) * el))
        local.bank = P.ExpertBank(*(None if t is None else t.detach().clone().requires_grad_()
                                    for t in (local.bank.up, local.bank.down, local.bank.bias_up, local.bank.bias_down)),
                                  first=rank * el)
        x = torch.randn(n, h, device="cuda", generator=torch.Generator(device="cuda").manual_seed(5)).bfloat16()
        x.requires_grad_()
        wd = P.World(1, world)
        g = P.ProcessGroup(P.EP, tuple(range(world)))
        ebr = [local.bank if r == rank else None for r in range(world)]
        drop = float(os.environ.get("_TEST_DROPOUT", "0"))
        ov = _test_override(n, k, e) if os.environ.get("_TEST_OVERRIDE") else None
        out, l_aux = P.ppmoe_forward(wd, g, x, local.gate, ebr, top_k=k, capacity_factor=cf, check_replicas=True,
                                     dropout_p=drop, rng=P.Rng(41, 2) if drop else None, route_override=ov)
        (out.float().sum() + l_aux).backward()
        P.sync_gate_gradients(wd, g, local.gate)
        torch.cuda.synchronize()
        res = {"out": out.detach().float().cpu().numpy(), "dx": x.grad.float().cpu().numpy(),
               "dwg": local.gate.wg.grad.cpu().numpy(), "dup": local.bank.up.grad.float().cpu().numpy(),
               "dbd": local.bank.bias_down.grad.float().cpu().numpy(), "l_aux": float(l_aux.detach()),
               "ar": wd.ledger.count_for("EP", "all_reduce"), "gs": wd.ledger.count_for("EP", "gradient_sync")}
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,k,cf,env,e", [(2, 2, float("inf"), {}, 2), (4, 2, 1.25, {}, 4), (4, 1, 1.0, {}, 4)])
def test_tp_one_expert_per_rank(world, k, cf, env, e):
    """E = T: one expert per rank (the C2 layout at T = 8), single-group GEMMs and the
    exchange with E < 8 gate columns."""
    test_tp_nccl_matches_simulated(world, k, cf, env, e)


@pytest.mark.parametrize("world,k,cf,env", [
    (2, 2, float("inf"), {}), (2, 1, 1.0, {}), (4, 2, 1.25, {}),
    (2, 2, 1.25, {"PPMOE_NVL_FWD": "fused"}), (2, 2, float("inf"), {"PPMOE_NVL_FWD": "slots"}),
    (2, 2, float("inf"), {"PPMOE_TP_COMM": "nccl"}), (2, 2, float("inf"), {"PPMOE_NVL_PUSH": "1", "PPMOE_NVL_PULL": "sm"}),
    (2, 2, float("inf"), {"PPMOE_NVL_MC": "1"}), (2, 2, 1.25, {"PPMOE_NVL_CHUNKS": "2"}),
    (2, 2, 1.25, {"_TEST_DROPOUT": "0.2"}), (4, 1, float("inf"), {"_TEST_DROPOUT": "0.1"}),
    (4, 2, float("inf"), {"PPMOE_NVL_CHUNKS": "2"}),
    (4, 2, 1.25, {"_TEST_N": "1022"}),  # N % T != 0: every rank routes the whole batch, uneven owner blocks
    (2, 2, 1.25, {"_TEST_OVERRIDE": "1"}),  # route override through the sliced routing records
])
def test_tp_nccl_matches_simulated(world, k, cf, env, e=8):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    import paper_2304_11414_b200 as P

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + os.getpid() % 500
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, k, cf, env, e)) for r in range(world)]
    for p in procs:
        p.start()
    got = _collect(q, procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # single-process reference: simulated TP world on GPU 0
    h, n = 512, int((env or {}).get("_TEST_N", "1024"))
    full = P.MoeLayerWeights.random(h, e, seed=11, device="cuda")
    x = torch.randn(n, h, device="cuda", generator=torch.Generator(device="cuda").manual_seed(5)).bfloat16()
    x.requires_grad_()
    drop = float((env or {}).get("_TEST_DROPOUT", "0"))
    ov = _test_override(n, k, e) if (env or {}).get("_TEST_OVERRIDE") else None
    out, l_aux = P.ppmoe_forward(P.World(1, world), P.ProcessGroup(P.EP, tuple(range(world))), x, full.gate,
                                 full.shard(world), top_k=k, capacity_factor=cf, dropout_p=drop,
                                 rng=P.Rng(41, 2) if drop else None, route_override=ov)
    (out.float().sum() + l_aux).backward()
    ref_out = out.detach().float().cpu().numpy()

    def err(a, b):
        return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))

    el = e // world
    for r in range(world):
        res = got[r]
        assert err(res["out"], ref_out) < 2e-2
        assert err(res["dx"], x.grad.float().cpu().numpy()) < 2e-2
        assert err(res["dwg"], full.gate.wg.grad.cpu().numpy()) < 2e-2
        assert err(res["dup"], full.bank.up.grad[r * el:(r + 1) * el].float().cpu().numpy()) < 2e-2
        assert err(res["dbd"], full.bank.bias_down.grad[r * el:(r + 1) * el].float().cpu().numpy()) < 2e-2
        assert abs(res["l_aux"] - float(l_aux.detach())) < 1e-5
        assert res["ar"] == 2 and res["gs"] == 1
    # every rank holds the identical replicated output, input gradient and synced gate
    # gradient (the peer-memory sums run in rank order on every rank)
    for r in range(1, world):
        assert np.array_equal(got[0]["out"], got[r]["out"])
        assert np.array_equal(got[0]["dx"], got[r]["dx"])
        assert np.array_equal(got[0]["dwg"], got[r]["dwg"])


def _dp_worker(rank, world, port, q, k, cf):
    import torch.distributed as dist

    import paper_2304_11414_b200 as P

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        h, e, n = 512, 8, 1024
        el = e // world
        full = P.MoeLayerWeights.random(h, e, seed=11, device="cuda")
        gate = P.GateParams(full.gate.wg.detach().clone().requires_grad_())
        bank = P.ExpertBank(*(None if t is None else t.detach().clone()[rank * el:(rank + 1) * el].contiguous().requires_grad_()
                              for t in (full.bank.up, full.bank.down, full.bank.bias_up, full.bank.bias_down)),
                            first=rank * el)
        xall = torch.randn(n, h, device="cuda", generator=torch.Generator(device="cuda").manual_seed(5)).bfloat16()
        nr = n // world
        x = xall[rank * nr:(rank + 1) * nr].clone().requires_grad_()
        wd = P.World(1, world)
        g = P.ProcessGroup(P.EP, tuple(range(world)))
        ebr = [bank if r == rank else None for r in range(world)]
        out, l_aux = P.dpmoe_forward(wd, g, x, gate, experts_by_rank=ebr, top_k=k, capacity_factor=cf)
        out.float().sum().backward()  # weight path only: aux terms differ between spans
        P.dpmoe_sync_gradients(wd, g, gate)
        torch.cuda.synchronize()
        q.put((rank, {"out": out.detach().float().cpu().numpy(), "dx": x.grad.float().cpu().numpy(),
                      "dwg": gate.wg.grad.cpu().numpy(), "dup": bank.up.grad.float().cpu().numpy(),
                      "a2a": wd.ledger.count_for("EP", "all_to_all")}))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,k,cf", [(2, 2, float("inf")), (2, 1, 0.9)])
def test_a2a_comparator_matches_ppmoe_on_global_batch(world, k, cf):
    """DPMoE over the ranks' micro-batches == PPMoE over their concatenation (same global
    capacity order), for outputs, dX and all weight gradients (moe.py:363-469 vs 254-308)."""
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    import paper_2304_11414_b200 as P

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + os.getpid() % 500
    procs = [ctx.Process(target=_dp_worker, args=(r, world, port, q, k, cf)) for r in range(world)]
    for p in procs:
        p.start()
    got = _collect(q, procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    h, e, n = 512, 8, 1024
    full = P.MoeLayerWeights.random(h, e, seed=11, device="cuda")
    x = torch.randn(n, h, device="cuda", generator=torch.Generator(device="cuda").manual_seed(5)).bfloat16()
    x.requires_grad_()
    out, _ = P.ppmoe_forward(P.World(1, 1), P.ProcessGroup(P.EP, (0,)), x, full.gate, [full.bank], top_k=k,
                             capacity_factor=cf)
    out.float().sum().backward()

    def err(a, b):
        return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))

    nr, el = n // world, e // world
    for r in range(world):
        res = got[r]
        assert err(res["out"], out.detach().float().cpu().numpy()[r * nr:(r + 1) * nr]) < 2e-2
        assert err(res["dx"], x.grad.float().cpu().numpy()[r * nr:(r + 1) * nr]) < 2e-2
        assert err(res["dwg"], full.gate.wg.grad.cpu().numpy()) < 2e-2
        assert err(res["dup"], full.bank.up.grad[r * el:(r + 1) * el].float().cpu().numpy()) < 2e-2
        assert res["a2a"] == 5


def _feed_worker(rank, world, port, q):
    import torch.distributed as dist

    import paper_2304_11414_b200 as P

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        n, h = 1024, 384
        hosts = [torch.randn(n, h, generator=torch.Generator().manual_seed(s)).bfloat16().pin_memory() for s in range(3)]
        feed = P.ReplicatedFeed(P.World(1, world), P.ProcessGroup(P.EP, tuple(range(world))), (n, h),
                                torch.bfloat16, "cuda")
        ok = []
        feed.submit(hosts[0])
        for i in range(3):
            x = feed.take()
            if i + 1 < 3:
                feed.submit(hosts[i + 1])
            ok.append(bool(torch.equal(x.cpu(), hosts[i])))
            torch.cuda.synchronize()
        q.put((rank, {"ok": ok, "h2d": feed.h2d_bytes}))
    finally:
        dist.destroy_process_group()


def test_replicated_feed_rebuilds_batch():
    """Each rank copies 1/T of the host batch; the all_gather replicates it exactly."""
    world = 2
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29800 + os.getpid() % 100
    procs = [ctx.Process(target=_feed_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = _collect(q, procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for r in range(world):
        assert got[r]["ok"] == [True, True, True]
        assert got[r]["h2d"] == 1024 * 384 * 2 // world


def _pp_worker(rank, world, port, q, stages, tp, dtype):
    import torch.distributed as dist

    import paper_2304_11414_b200 as P
    from paper_2304_11414_b200.pipeline import PipelineStack, schedule_1f1b

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        stack = PipelineStack(P.World(1, world), layers=4, stages=stages, tp=tp, hidden=256, experts=8, top_k=2,
                              seed=3, dtype=dtype)
        done = stack.train_step(3, mb_tokens=384)
        stack.sync_gate_gradients()
        torch.cuda.synchronize()
        grads = {}
        for j, (dense, moe) in enumerate(stack.blocks):
            li = stack.first_layer + j
            grads[f"{li}.dense.up"] = dense.up.grad.float().cpu().numpy()
            grads[f"{li}.moe.wg"] = moe.gate.wg.grad.cpu().numpy()
            grads[f"{li}.moe.up"] = moe.bank.up.grad.float().cpu().numpy()
        q.put((rank, {"done": done, "expected": schedule_1f1b(stages, 3)[stack.stage], "grads": grads,
                      "stage": stack.stage, "slot": stack.slot}))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("stages,tp,dtype", [(2, 1, torch.bfloat16), (2, 2, torch.float32),
                                             (2, 4, torch.float32)])  # 2 x 4: BASELINE configs[3] on 8 GPUs
def test_pipeline_stack_matches_single_gpu(stages, tp, dtype):
    """1F1B over P stages x T tensor ranks (NCCL p2p, TP dense FFN, PPMoE exchange) gives the
    gradients of the same 4-block stack run on one GPU (BASELINE configs[3] structure).
    With T = 1 the arithmetic is identical (bf16); with T = 2 the sharded dense FFN
    changes bf16 rounding and, through routing near-ties amplified by the residual stack,
    whole tokens' gradients, so the tensor-parallel composition is checked in fp32."""
    world = stages * tp
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    import paper_2304_11414_b200 as P
    from paper_2304_11414_b200.pipeline import PipelineStack

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29900 + os.getpid() % 90
    procs = [ctx.Process(target=_pp_worker, args=(r, world, port, q, stages, tp, dtype)) for r in range(world)]
    for p in procs:
        p.start()
    got = _collect(q, procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ref = PipelineStack(P.World(1, 1), layers=4, stages=1, tp=1, hidden=256, experts=8, top_k=2, seed=3, dtype=dtype)
    ref.train_step(3, mb_tokens=384)
    torch.cuda.synchronize()

    def err(a, b):
        return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))

    el, fs = 8 // tp, 1024 // tp
    for r in range(world):
        res = got[r]
        assert res["done"] == res["expected"]
        t = res["slot"]
        for key, g in res["grads"].items():
            li, part, name = key.split(".")
            dense, moe = ref.blocks[int(li)]
            if part == "dense":
                want = dense.up.grad[:, t * fs:(t + 1) * fs].float().cpu().numpy()
            elif name == "wg":
                want = moe.gate.wg.grad.cpu().numpy()
            else:
                want = moe.bank.up.grad[t * el:(t + 1) * el].float().cpu().numpy()
            assert err(g, want) < (3e-2 if dtype == torch.bfloat16 else 1e-3), (key, err(g, want))


def _full_worker(rank, world, port, q, cfg):
    """One rank of a BASELINE-size layer on BASELINE's inputs (Rng(0) weights, this rank's
    expert block only; Rng(1, 99) hidden).  The fp64 reference is the same TP decomposition
    in fp64: this rank's experts give partial out / dX / dS, summed over the group by an
    fp64 NCCL all-reduce, then the gate backward (ppmoe_testlib.fp64_*)."""
    import json

    import torch.distributed as dist

    import paper_2304_11414_b200 as P
    from oracle import ppmoe_oracle as O
    from ppmoe_testlib import dev_scaled_err, fp64_expert_pass, fp64_gate_pass, routing_on_device

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        h, e, k, cf = {"C2": (4096, 8, 2, float("inf")), "C3": (8192, 16, 2, 1.25)}[cfg]
        n = 16384
        el = e // world
        ids = range(rank * el, (rank + 1) * el)
        w = P.MoeLayerWeights.init(h, e, P.Rng(0), device="cuda", experts=ids,
                                   threads=max(1, (os.cpu_count() or 1) // world))
        x = P.Rng(1, 99).normal_tensor((n, h), dtype=torch.bfloat16).requires_grad_()
        wd = P.World(1, world)
        g = P.ProcessGroup(P.EP, tuple(range(world)))
        out, l_aux = P.ppmoe_forward(wd, g, x, w.gate, [w.bank if r == rank else None for r in range(world)],
                                     top_k=k, capacity_factor=cf, check_replicas=True)
        torch.autograd.backward([out, l_aux], [torch.ones_like(out), torch.ones_like(l_aux)])
        P.sync_gate_gradients(wd, g, w.gate)
        torch.cuda.synchronize()
        x64 = x.detach().double().cpu().numpy()
        wg64 = w.gate.wg.detach().double().cpu().numpy()
        route = O.gate_topk(x64, wg64, k)
        _, kept, _ = O.dispatch_plan(route.indices, e, O.capacity_of(cf, n, k, e))
        idx, wts, kept_d, scores, cnt = routing_on_device(route, kept)
        errs = {}
        ours = {"up": w.bank.up.grad, "down": w.bank.down.grad, "bias_up": w.bank.bias_up.grad,
                "bias_down": w.bank.bias_down.grad}

        def on_expert(ex, grads):
            for nm, gr in grads.items():
                errs[f"expert{ex}.{nm}"] = dev_scaled_err(ours[nm][ex - ids[0]], gr)

        with torch.no_grad():
            out_r, dx_r, ds = fp64_expert_pass(x, w.bank, list(ids), idx, wts, kept_d, e, on_expert=on_expert)
            for t in (out_r, dx_r, ds):
                dist.all_reduce(t)
            errs["out"] = dev_scaled_err(out, out_r)
            dwg_r, dxg = fp64_gate_pass(x, w.gate.wg, scores, cnt, ds)
            errs["grad_hidden"] = dev_scaled_err(x.grad, dx_r + dxg)
            errs["gate.wg"] = dev_scaled_err(w.gate.wg.grad, dwg_r)
        print(json.dumps({"cfg": cfg, "tp": world, "rank": rank, "errors": errs}), flush=True)
        res = {"errs": errs, "l_aux": abs(float(l_aux.detach()) - route.l_aux),
               "digest": float(out.detach().float().sum()), "ndrop": int((~kept).sum())}
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg,world", [("C2", 2), ("C2", 4), ("C3", 2), ("C3", 4)])
def test_tp_full_size_every_gradient(cfg, world):
    """BASELINE configs[1] / configs[2] at full size over the NVLink exchange (T = 2, 4) on
    BASELINE's inputs: the replicated out and dX, the synced dWg and every local expert
    gradient over every element against the fp64 closed form, on every rank."""
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + (os.getpid() + 7 * world + len(cfg)) % 500
    procs = [ctx.Process(target=_full_worker, args=(r, world, port, q, cfg)) for r in range(world)]
    for p in procs:
        p.start()
    got = _collect(q, procs, timeout=900)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    e = {"C2": 8, "C3": 16}[cfg]
    for r in range(world):
        errs = got[r]["errs"]
        bad = {key: v for key, v in errs.items() if not v < 2e-2}
        assert not bad and got[r]["l_aux"] < 1e-5, (r, bad, got[r]["l_aux"])
        assert len(errs) == 3 + 4 * (e // world)
    assert len({got[r]["digest"] for r in range(world)}) == 1  # identical replicas


def _barrier_timeout_worker(rank, world, port, q):
    """Rank 1 enters a barrier its peer never joins: the barrier times out, the arena's
    host-mapped flag is set, and both the explicit check and the next layer call raise."""
    os.environ["PPMOE_NVL_TIMEOUT_CYCLES"] = "200000000"  # ~0.1-0.15 s
    import torch.distributed as dist

    import paper_2304_11414_b200 as P
    from paper_2304_11414_b200 import nvlink

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        wd = P.World(1, world)
        g = P.ProcessGroup(P.EP, tuple(range(world)))
        assert nvlink.enabled(wd, g, torch.bfloat16, 256)
        ar = nvlink.arena(wd, g)
        res = {"raised_check": False, "raised_forward": False}
        if rank == 1:
            ar.barrier(3)  # rank 0 never arrives on channel 3
            try:
                ar.check()
            except RuntimeError as exc:
                res["raised_check"] = "timed out" in str(exc)
            w = P.MoeLayerWeights.random(256, 4, seed=1, device="cuda", experts=range(2, 4))
            x = torch.randn(64, 256, device="cuda").bfloat16()
            try:
                P.ppmoe_forward(wd, g, x, w.gate, [None, w.bank], top_k=2)
            except RuntimeError as exc:
                res["raised_forward"] = "timed out" in str(exc)
        torch.cuda.synchronize()
        q.put((rank, res))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_nvl_barrier_timeout_raises():
    """A peer that skips a barrier makes the exchange fail loudly: the timed-out
    barrier's flag is read from pinned host memory and ppmoe_forward raises RuntimeError."""
    world = 2
    if torch.cuda.device_count() < world:
        pytest.skip("needs 2 GPUs")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + (os.getpid() + 13) % 500
    procs = [ctx.Process(target=_barrier_timeout_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = _collect(q, procs, timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert got[1]["raised_check"] and got[1]["raised_forward"], got[1]
    assert not got[0]["raised_check"] and not got[0]["raised_forward"]


def _divergence_worker(rank, world, port, q):
    """Identical hidden, different route overrides per rank (full routing on every rank, no
    sliced router): check_replicas must report the dispatch divergence (moe.py:289-291)."""
    os.environ["PPMOE_SLICED_ROUTER"] = "0"
    import torch.distributed as dist

    import paper_2304_11414_b200 as P

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        w = P.MoeLayerWeights.random(256, 4, seed=3, device="cuda", experts=range(2 * rank, 2 * rank + 2))
        x = torch.randn(64, 256, device="cuda", generator=torch.Generator(device="cuda").manual_seed(4)).bfloat16()
        wd, g = P.World(1, world), P.ProcessGroup(P.EP, (0, 1))
        ebr = [w.bank if r == rank else None for r in range(world)]
        ok_same = True
        try:  # same routing everywhere: no error
            P.ppmoe_forward(wd, g, x, w.gate, ebr, top_k=1, check_replicas=True)
        except ValueError:
            ok_same = False
        ov = torch.full((64,), rank, dtype=torch.int64, device="cuda")  # rank 0 -> expert 0, rank 1 -> 1
        msg = ""
        try:
            P.ppmoe_forward(wd, g, x, w.gate, ebr, top_k=1, route_override=ov, check_replicas=True)
        except ValueError as exc:
            msg = str(exc)
        torch.cuda.synchronize()
        q.put((rank, {"ok_same": ok_same, "msg": msg}))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_check_replicas_detects_dispatch_divergence():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + (os.getpid() + 17) % 500
    procs = [ctx.Process(target=_divergence_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = _collect(q, procs, timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for r in range(2):
        assert got[r]["ok_same"], got[r]
        assert "dispatch order differs" in got[r]["msg"], got[r]
