"""Where the end-to-end call's time goes (C4, 4096 poses, 640x480): host wall clock of
hp_eval_costs_host vs the device time of its launches, with and without zero-copy, and a
device-resident call.   python scripts/e2e_probe.py"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2005_07068_b200 as hp  # noqa: E402
import workloads as W  # noqa: E402


def main():
    ctx = hp.Context(640, 480, max_particles=4096)
    d, m = ctx.render_observation(W.H_A)
    ctx.set_observation(d, m)
    sw = W.swarm_c4().astype(np.float32)
    pin_in = torch.from_numpy(sw).pin_memory()
    pin_out = torch.empty(4096, dtype=torch.float32).pin_memory()
    hin, hout = pin_in.numpy(), pin_out.numpy()
    P = torch.tensor(sw, device="cuda")
    C = torch.empty(4096, device="cuda")
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    for name, fn in (("host (zero-copy)", lambda: ctx.eval_costs_host(hin, out=hout)),
                     ("device + sync", lambda: (ctx.eval_costs(P, out=C), torch.cuda.synchronize()))):
        for _ in range(20):
            fn()
        ctx.set_timing(True)
        ts, ks = [], []
        for _ in range(100):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
            ks.append(sum(ctx.last_kernel_ms()))
        ctx.set_timing(False)
        ts = np.array(ts) * 1e3
        print(f"{name:18s} wall {np.median(ts):.4f} ms  kernels {np.median(ks):.4f} ms  "
              f"overhead {np.median(ts) - np.median(ks):.4f} ms")
    t0 = time.perf_counter()
    for _ in range(1000):
        ctx.splits_for(4096)
    print(f"ctypes call        {(time.perf_counter() - t0):.4f} us")


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def floor_probe():
    """Launch + sync floor of this box: a tiny torch kernel, and hp calls split into
    launch-only (no sync) and sync."""
    x = torch.zeros(1, device="cuda")
    for _ in range(100):
        x.add_(1)
        torch.cuda.synchronize()
    ts = []
    for _ in range(200):
        t0 = time.perf_counter()
        x.add_(1)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(f"tiny kernel + sync  {np.median(ts) * 1e6:.1f} us")
    ctx = hp.Context(640, 480, max_particles=4096)
    d, m = ctx.render_observation(W.H_A)
    ctx.set_observation(d, m)
    P = torch.tensor(W.swarm_c4().astype(np.float32), device="cuda")
    C = torch.empty(4096, device="cuda")
    for _ in range(20):
        ctx.eval_costs(P, out=C)
    torch.cuda.synchronize()
    tl, tsy = [], []
    for _ in range(100):
        t0 = time.perf_counter()
        ctx.eval_costs(P, out=C)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        tl.append(t1 - t0)
        tsy.append(t2 - t0)
    print(f"hp eval launch-only {np.median(tl) * 1e6:.1f} us, launch+sync {np.median(tsy) * 1e6:.1f} us")


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "floor":
    floor_probe()


def tiny_probe():
    """Host-path floor: hp_eval_costs_host / hp_eval_costs on 1 and 64 poses."""
    ctx = hp.Context(640, 480, max_particles=4096)
    d, m = ctx.render_observation(W.H_A)
    ctx.set_observation(d, m)
    sw = W.swarm_c4().astype(np.float32)
    pin_in = torch.from_numpy(sw).pin_memory()
    pin_out = torch.empty(4096, dtype=torch.float32).pin_memory()
    P = torch.tensor(sw, device="cuda")
    C = torch.empty(4096, device="cuda")
    for n in (1, 64, 4096):
        hin, hout = pin_in.numpy()[:n], pin_out.numpy()[:n]
        for name, fn in (("host", lambda: ctx.eval_costs_host(hin, out=hout)),
                         ("device+sync", lambda: (ctx.eval_costs(P[:n], out=C[:n]),
                                                  torch.cuda.synchronize()))):
            for _ in range(20):
                fn()
            ts = []
            for _ in range(200):
                t0 = time.perf_counter()
                fn()
                ts.append(time.perf_counter() - t0)
            print(f"n={n:5d} {name:12s} {np.median(ts) * 1e6:8.1f} us")


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "tiny":
    tiny_probe()
