"""H2D copy bandwidth from pinned host memory with the host idle vs with N busy host
processes (uncore frequency scaling check).  usage: python tools/h2d_uncore_probe.py"""
import json
import multiprocessing as mp
import time

import torch


def spin(stop):
    x = 0
    while not stop.is_set():
        x += 1


def h2d_ms(src, dst, reps=20):
    out = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dst.copy_(src, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
        time.sleep(0.01)
    out.sort()
    return out[len(out) // 2]


if __name__ == "__main__":
    n = 75 << 20
    src = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    src.fill_(1)
    dst = torch.empty(n, dtype=torch.uint8, device="cuda")
    h2d_ms(src, dst, 3)
    for busy in (0, 1, 4, 16):
        stop = mp.Event()
        ps = [mp.Process(target=spin, args=(stop,)) for _ in range(busy)]
        for p in ps:
            p.start()
        time.sleep(0.2)
        ms = h2d_ms(src, dst)
        stop.set()
        for p in ps:
            p.join()
        print(json.dumps({"busy_procs": busy, "h2d_ms_75MB": ms, "GBps": n / ms / 1e6}), flush=True)
