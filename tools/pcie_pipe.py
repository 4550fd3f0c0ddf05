"""Diagnostics: the e2e copy pattern of scan2d_train_host without kernels --
cfg2's 128 scans in the library's chunk schedule (ramped first / last chunk),
5 host->device copies per piece on one stream, 5 device->host copies on
another, each piece's D2H after its H2D (an event), three rotating slots."""
import time
import torch

S, H, W, N = 128, 200, 200, 16
hw = H * W
sizes = [2, 2, 4, 8] + [16] * 6 + [8, 4, 2, 2]
assert sum(sizes) == S
per_in = [hw, hw, hw * N, hw * N, hw]
hin = [torch.empty(S * n, dtype=torch.float32).pin_memory() for n in per_in]
hout = [torch.empty(S * n, dtype=torch.float32).pin_memory() for n in per_in]
slots = [[torch.empty(16 * n, device="cuda") for n in per_in] for _ in range(3)]
h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()


def step(kernel_us=0):
    free = [None] * 3
    s0 = 0
    for k, sk in enumerate(sizes):
        sl = slots[k % 3]
        with torch.cuda.stream(h2d):
            if free[k % 3] is not None:
                h2d.wait_event(free[k % 3])
            for i, n in enumerate(per_in):
                sl[i][: sk * n].copy_(hin[i][s0 * n:(s0 + sk) * n], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(h2d)
        with torch.cuda.stream(d2h):
            d2h.wait_event(ev)
            if kernel_us:
                torch.cuda._sleep(int(kernel_us * 1900))
            for i, n in enumerate(per_in):
                hout[i][s0 * n:(s0 + sk) * n].copy_(sl[i][: sk * n], non_blocking=True)
            fe = torch.cuda.Event()
            fe.record(d2h)
            free[k % 3] = fe
        s0 += sk
    torch.cuda.synchronize()


for kus in (0, 60):
    step(kus)
    t0 = time.perf_counter()
    for _ in range(5):
        step(kus)
    dt = (time.perf_counter() - t0) / 5
    byts = sum(S * n * 4 for n in per_in)
    print(f"kernel {kus} us/piece: {dt * 1e3:.2f} ms per step, {byts / dt / 1e9:.1f} GB/s each way, "
          f"{S * hw / dt / 1e9:.3f} Gelem/s")
