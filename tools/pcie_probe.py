"""PCIe copy bandwidth on the GPU box: pinned H2D, D2H, both at once, and
chunked / multi-stream variants (the e2e leg of bench.py is copy-bound).

    python tools/pcie_probe.py
"""
import time

import torch


def bw(fn, nbytes, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return nbytes / best / 1e9, best * 1e3


def main():
    dev = torch.device("cuda", 0)
    nb = 1_233_097_296
    h_in = torch.empty(nb, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(nb, dtype=torch.uint8).pin_memory()
    d_in = torch.empty(nb, dtype=torch.uint8, device=dev)
    d_out = torch.empty(nb, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def h2d():
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)

    def both():
        h2d()
        d2h()

    def h2d_chunks(k):
        def f():
            streams = [torch.cuda.Stream() for _ in range(k)]
            step = (nb + k - 1) // k
            for i, s in enumerate(streams):
                with torch.cuda.stream(s):
                    d_in[i * step:(i + 1) * step].copy_(h_in[i * step:(i + 1) * step], non_blocking=True)
        return f

    print("h2d      %.1f GB/s (%.1f ms)" % bw(h2d, nb))
    print("d2h      %.1f GB/s (%.1f ms)" % bw(d2h, nb))
    g, ms = bw(both, 2 * nb)
    print("both     %.1f GB/s aggregate (%.1f ms for 2 x %.2f GB)" % (g, ms, nb / 1e9))
    for k in (2, 4):
        print(f"h2d x{k} streams %.1f GB/s (%.1f ms)" % bw(h2d_chunks(k), nb))
    print(torch.cuda.get_device_name(0))


if __name__ == "__main__":
    main()
