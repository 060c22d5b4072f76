#!/usr/bin/env python
"""PCIe floor of bench.py's e2e step: the 19 operators' u vectors up and y
vectors down (pinned host buffers of the bench's sizes), as bare copies --
H2D only, D2H only, and both directions concurrently on two streams -- plus
the host topology (NUMA nodes, GPU locality).  Explains how far the host
entry's ~65-75 ms per step is from what the link can do."""
import glob
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

import bench


def sh(cmd):
    try:
        return subprocess.run(cmd, shell=True, capture_output=True, text=True, timeout=20).stdout.strip()
    except Exception as e:  # noqa: BLE001
        return f"({e})"


def main():
    print("# lscpu:", sh("lscpu | grep -E 'NUMA|Socket|Model name|^CPU\\(s\\)' | tr '\\n' ';'"))
    print("# affinity:", len(os.sched_getaffinity(0)), sorted(os.sched_getaffinity(0))[:4], "...")
    for f in glob.glob("/sys/bus/pci/devices/*/numa_node"):
        dev = os.path.dirname(f)
        try:
            if open(os.path.join(dev, "vendor")).read().strip() == "0x10de":
                print("# gpu", os.path.basename(dev), "numa_node", open(f).read().strip())
        except OSError:
            pass
    print("# topo:", sh("nvidia-smi topo -m | head -6 | tr '\\n' ';'"))
    sizes = [bench.op_meta(n)["dofs"] for n in bench.BASELINE_OPS]
    hu = [torch.empty(n, dtype=torch.float64, pin_memory=True).fill_(1.0) for n in sizes]
    hy = [torch.empty(n, dtype=torch.float64, pin_memory=True) for n in sizes]
    du = [torch.empty(n, dtype=torch.float64, device="cuda") for n in sizes]
    dy = [torch.zeros(n, dtype=torch.float64, device="cuda") for n in sizes]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    gb = 8e-9 * sum(sizes)

    def up():
        with torch.cuda.stream(s1):
            for d, h in zip(du, hu):
                d.copy_(h, non_blocking=True)

    def down():
        with torch.cuda.stream(s2):
            for h, d in zip(hy, dy):
                h.copy_(d, non_blocking=True)

    def t(fn, reps=5):
        best = 1e9
        for _ in range(reps + 1):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        return best

    r = {"gb_each_way": gb, "h2d_ms": 1e3 * t(up), "d2h_ms": 1e3 * t(down),
         "duplex_ms": 1e3 * t(lambda: (up(), down()))}
    r["h2d_gbs"] = gb / r["h2d_ms"] * 1e3
    r["d2h_gbs"] = gb / r["d2h_ms"] * 1e3
    r["duplex_gbs_total"] = 2 * gb / r["duplex_ms"] * 1e3
    print(json.dumps(r))


if __name__ == "__main__":
    main()
