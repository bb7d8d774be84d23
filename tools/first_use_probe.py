"""Which host calls wait for another stream's running kernel?

A thread keeps a long kernel (torch.cuda._sleep) running on stream A; the
main thread then issues, on stream B, the torch ops the co-resident tests
use between two exchanges -- each for the first time in the process, then
again -- and prints each call's host time.  A call that takes ~the sleep
kernel's remaining time waited for it: on a GPU hosting several ranks of
one comm, such a call stalls every peer rank's engine (they spin on this
rank's next exchange) until their timeout.

  python tools/first_use_probe.py            (CUDA_MODULE_LOADING as set)
"""
import os
import threading
import time

import torch


def main():
    torch.cuda.set_device(0)
    a, b = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(b):
        x = torch.randn(777, 96, device="cuda")
        order = torch.randperm(1554, device="cuda")
        w = torch.rand(777, 2, device="cuda")
        torch.cuda.synchronize()

    def spin(seconds):
        with torch.cuda.stream(a):
            torch.cuda._sleep(int(seconds * 1.9e9))

    ops = [
        ("zeros", lambda: torch.zeros(777, 96, device="cuda")),
        ("floordiv", lambda: order // 2),
        ("index", lambda: w.reshape(-1)[order]),
        ("mul", lambda: x * 2.0),
        ("index_add_", lambda: torch.zeros(777, 96, device="cuda").index_add_(0, order // 2, x.repeat(2, 1))),
        ("argsort", lambda: torch.argsort(order, stable=True)),
        ("bincount", lambda: torch.bincount(order % 7, minlength=8)),
        ("index_select", lambda: torch.index_select(x, 0, order[:700] // 2)),
        ("where", lambda: torch.where(order > 5, order, torch.zeros_like(order))),
        ("randint", lambda: torch.randint(0, 16, (777, 2), device="cuda")),
        ("allclose", lambda: torch.allclose(x, x)),
        ("tolist", lambda: order[:8].tolist()),
        ("empty_4g", lambda: torch.empty(4 << 30, dtype=torch.uint8, device="cuda")),
    ]
    print(f"CUDA_MODULE_LOADING={os.environ.get('CUDA_MODULE_LOADING')}")
    for rnd in ("first", "again"):
        for name, fn in ops:
            t = threading.Thread(target=spin, args=(2.0,))
            t.start()
            time.sleep(0.3)  # the sleep kernel is running on stream A
            with torch.cuda.stream(b):
                t0 = time.perf_counter()
                fn()
                dt = time.perf_counter() - t0
            t.join()
            torch.cuda.synchronize()
            print(f"{rnd:5s} {name:12s} host {dt * 1e3:9.2f} ms{'   <-- waited' if dt > 0.5 else ''}", flush=True)


if __name__ == "__main__":
    main()
