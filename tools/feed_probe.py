"""Dev tool: host->device feed timing at the C2 shape (single GPU)."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2304_11414_b200 as P

n, h = 16384, 4096
dev = torch.device("cuda", 0)
x_host = torch.randn(n, h).to(torch.bfloat16).pin_memory()
print("pinned", x_host.is_pinned(), x_host[0:n].is_pinned())
x_dev = torch.empty(n, h, device=dev, dtype=torch.bfloat16)


def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


print("copy default stream ms", t(lambda: x_dev.copy_(x_host, non_blocking=True)))
s = torch.cuda.Stream()
def side():
    with torch.cuda.stream(s):
        x_dev.copy_(x_host, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s)
print("copy side stream ms", t(side))
feed = P.ReplicatedFeed(P.World(1, 1), P.ProcessGroup(P.EP, (0,)), (n, h), torch.bfloat16, dev)
def fd():
    feed.submit(x_host)
    feed.take()
print("feed submit+take ms", t(fd))
w = P.MoeLayerWeights.random(h, 8, seed=0, device=dev)
g_out = torch.ones(n, h, device=dev, dtype=torch.bfloat16)
def step(xin):
    out, l_aux = P.ppmoe_forward(P.World(1, 1), P.ProcessGroup(P.EP, (0,)), xin, w.gate, [w.bank], top_k=2)
    torch.autograd.backward([out, l_aux], [g_out, torch.ones((), device=dev)])
    return out, l_aux
xr = x_dev.detach().requires_grad_()
print("step ms", t(lambda: step(xr)))
def e2e_old():
    x_dev.copy_(x_host, non_blocking=True)
    step(x_dev.detach().requires_grad_())
print("copy+step ms", t(e2e_old))
def e2e_new(steps=10):
    feed.submit(x_host)
    for i in range(steps):
        xin = feed.take().detach().requires_grad_()
        if i + 1 < steps:
            feed.submit(x_host)
        step(xin)
print("feed loop of 10, per step ms", t(lambda: e2e_new(), reps=1) / 10)
loss_host = torch.empty(1, dtype=torch.float32).pin_memory()
def e2e_sync(steps=10, use_feed=True):
    if use_feed:
        feed.submit(x_host)
    for i in range(steps):
        if use_feed:
            xin = feed.take().detach().requires_grad_()
            if i + 1 < steps:
                feed.submit(x_host)
        else:
            x_dev.copy_(x_host, non_blocking=True)
            xin = x_dev.detach().requires_grad_()
        out, l_aux = step(xin)
        loss = out.float().sum() + l_aux
        loss_host.copy_(loss.reshape(1), non_blocking=True)
        torch.cuda.current_stream().synchronize()
        float(loss_host[0])
for uf in (False, True, False, True):
    t0 = time.perf_counter()
    ms = t(lambda: e2e_sync(use_feed=uf), reps=1) / 10
    print("bench-style e2e feed=", uf, "per step ms", ms, "wall", (time.perf_counter() - t0) / 20 * 1e3)
