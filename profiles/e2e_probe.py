"""Where does the e2e step's time go? PCIe copy bandwidth (pinned, one and
several streams, duplex) against the e2e step (3 tcb_run calls with host
buffers) issued serially, from 3 threads, and asynchronously on 3 streams."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1802_04730_b200 import ExecutionEngine  # noqa: E402


def wall(fn, n=200, warm=20):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6


def gpu_local_cpus(index=0):
    """CPUs on the GPU's NUMA node (NVML CPU affinity mask), or None."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(index)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, 16)
        cpus = {w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1}
        return cpus & os.sched_getaffinity(0) or None
    except Exception:
        return None


def main():
    if os.environ.get("E2E_PIN_LOCAL") == "1":
        c = gpu_local_cpus()
        print("gpu-local cpus:", sorted(c)[:4], "...", len(c) if c else None, "of", os.cpu_count(), flush=True)
        if c:
            os.sched_setaffinity(0, c)
    dev = torch.device("cuda", 0)
    ss = [torch.cuda.Stream() for _ in range(4)]
    for mb in (1.5, 7.5, 8.85, 64):
        n = int(mb * 2**20 / 4)
        h = torch.empty(n, pin_memory=True)
        d = torch.empty(n, device=dev)

        def one():
            d.copy_(h, non_blocking=True)
        us = wall(one)
        print(f"H2D {mb:6.2f} MiB one stream      {us:8.1f} us  {n * 4 / us / 1e3:6.1f} GB/s", flush=True)

        def back():
            h.copy_(d, non_blocking=True)
        us = wall(back)
        print(f"D2H {mb:6.2f} MiB one stream      {us:8.1f} us  {n * 4 / us / 1e3:6.1f} GB/s", flush=True)

    # duplex: 7.5 MiB in while 1.5 MiB out on another stream
    hi = torch.empty(int(7.5 * 2**18), pin_memory=True)
    di = torch.empty(hi.numel(), device=dev)
    ho = torch.empty(int(1.5 * 2**18), pin_memory=True)
    do = torch.empty(ho.numel(), device=dev)

    def duplex():
        with torch.cuda.stream(ss[0]):
            di.copy_(hi, non_blocking=True)
        with torch.cuda.stream(ss[1]):
            ho.copy_(do, non_blocking=True)
    print(f"duplex 7.5 in + 1.5 out           {wall(duplex):8.1f} us", flush=True)

    # H2D split over 4 streams
    parts = [torch.empty(int(8.85 * 2**18) // 4, pin_memory=True) for _ in range(4)]
    dparts = [torch.empty(p.numel(), device=dev) for p in parts]

    def split4():
        for p, dp, s in zip(parts, dparts, ss):
            with torch.cuda.stream(s):
                dp.copy_(p, non_blocking=True)
    print(f"H2D 8.85 MiB over 4 streams       {wall(split4):8.1f} us", flush=True)

    ee = ExecutionEngine()
    ops = [bench.OpInstance(ee, torch, n, s, sd, 1, dev, 1 + i) for i, (n, s, sd) in enumerate(bench.STEP_OPS)]
    host = []
    for o in ops:
        ps, os_ = o.sets[0]
        hp = [x.cpu().pin_memory() for x in ps]
        ho = [x.cpu().pin_memory() for x in os_]
        host.append((o.name, ee.compile(o.name, hp, ho), hp, ho))
    for name, hh, hp, ho in host:
        us = wall(lambda: ee.run(hh, hp, ho, stream=ss[0].cuda_stream), n=100)
        nb = sum(x.numel() * 4 for x in hp)
        print(f"e2e {name:8s} alone              {us:8.1f} us  ({nb / 2**20:.2f} MiB in)", flush=True)

    def serial():
        for name, hh, hp, ho in host:
            ee.run(hh, hp, ho, stream=ss[0].cuda_stream)
    print(f"e2e step serial                   {wall(serial, n=100):8.1f} us", flush=True)

    import concurrent.futures as cf
    pool = cf.ThreadPoolExecutor(3)

    def one(j):
        name, hh, hp, ho = host[j]
        ee.run(hh, hp, ho, stream=ss[j].cuda_stream)

    def threads():
        list(pool.map(one, range(3)))
    print(f"e2e step 3 threads                {wall(threads, n=100):8.1f} us", flush=True)

    def asyn():
        for j, (name, hh, hp, ho) in enumerate(host):
            ee.run(hh, hp, ho, stream=ss[j].cuda_stream, sync=False)
        for j in range(3):
            ss[j].synchronize()
    print(f"e2e step async 3 streams          {wall(asyn, n=100):8.1f} us", flush=True)

    def asyn1():
        for j, (name, hh, hp, ho) in enumerate(host):
            ee.run(hh, hp, ho, stream=ss[0].cuda_stream, sync=False)
        ss[0].synchronize()
    print(f"e2e step async 1 stream           {wall(asyn1, n=100):8.1f} us", flush=True)

    prep = [ee.prepare(hh, hp, ho) for name, hh, hp, ho in host]
    for (name, hh, hp, ho), pr in zip(host, prep):
        us = wall(lambda: pr.run(stream=ss[0].cuda_stream), n=100)
        print(f"e2e {name:8s} prepared           {us:8.1f} us", flush=True)

    def prep3(order=(0, 1, 2)):
        for j in order:
            prep[j].run(stream=ss[j].cuda_stream, sync=False)
        for j in order:
            ss[j].synchronize()
    print(f"e2e step prepared async 3 streams {wall(prep3, n=200):8.1f} us", flush=True)
    print(f"e2e step prepared async, small 1st{wall(lambda: prep3((1, 2, 0)), n=200):8.1f} us", flush=True)


if __name__ == "__main__":
    main()
