"""Diagnostics: the e2e copy pattern of scan2d_train_host without kernels --
cfg2's 128 scans in chunk schedules (the library's ramped one and variants),
5 host->device copies per piece, 5 device->host copies per piece, each piece's
D2H after its H2D (an event), three rotating slots; `streams` copy streams per
direction used round-robin over pieces."""
import time
import torch

S, H, W, N = 128, 200, 200, 16
hw = H * W
per_in = [hw, hw, hw * N, hw * N, hw]
hin = [torch.empty(S * n, dtype=torch.float32).pin_memory() for n in per_in]
hout = [torch.empty(S * n, dtype=torch.float32).pin_memory() for n in per_in]
NSLOT = 4
slots = [[torch.empty(32 * n, device="cuda") for n in per_in] for _ in range(NSLOT)]


def run(sizes, streams=1, kernel_us=0):
    h2d = [torch.cuda.Stream() for _ in range(streams)]
    d2h = [torch.cuda.Stream() for _ in range(streams)]

    def step():
        free = [None] * NSLOT
        s0 = 0
        for k, sk in enumerate(sizes):
            sl = slots[k % NSLOT]
            hs, ds = h2d[k % streams], d2h[k % streams]
            with torch.cuda.stream(hs):
                if free[k % NSLOT] is not None:
                    hs.wait_event(free[k % NSLOT])
                for i, n in enumerate(per_in):
                    sl[i][: sk * n].copy_(hin[i][s0 * n:(s0 + sk) * n], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(hs)
            with torch.cuda.stream(ds):
                ds.wait_event(ev)
                if kernel_us:
                    torch.cuda._sleep(int(kernel_us * 1900))
                for i, n in enumerate(per_in):
                    hout[i][s0 * n:(s0 + sk) * n].copy_(sl[i][: sk * n], non_blocking=True)
                fe = torch.cuda.Event()
                fe.record(ds)
                free[k % NSLOT] = fe
            s0 += sk
        torch.cuda.synchronize()

    step()
    t0 = time.perf_counter()
    for _ in range(5):
        step()
    dt = (time.perf_counter() - t0) / 5
    return dt


byts = sum(S * n * 4 for n in per_in)
for name, sizes, st in [("library ramp 8 chunks", [2, 2, 4, 8] + [16] * 6 + [8, 4, 2, 2], 1),
                        ("8 chunks no ramp", [16] * 8, 1),
                        ("16 chunks", [8] * 16, 1),
                        ("ramp, 2 streams/dir", [2, 2, 4, 8] + [16] * 6 + [8, 4, 2, 2], 2),
                        ("32 chunks, 2 streams/dir", [4] * 32, 2),
                        ("fine ramp 1,1,2,4,8 + 8x14 + ...", [1, 1, 2, 4, 8] + [8] * 13 + [4, 2, 1, 1], 1)]:
    assert sum(sizes) == S, name
    dt = run(sizes, st)
    print(f"{name}: {dt * 1e3:.2f} ms, {byts / dt / 1e9:.1f} GB/s each way, {S * hw / dt / 1e9:.3f} Gelem/s")
