"""Host DRAM bandwidth on the GPU box (DESIGN 6: the per-GPU host budget of the
zero-copy window fetch against what the host memory system delivers). numpy
copies release the GIL, so T Python threads copy in parallel; read+write bytes."""
import json, os, threading, time
import numpy as np

def run(threads, mb=512, reps=4):
    bufs = [(np.ones(mb << 20, np.uint8), np.empty(mb << 20, np.uint8)) for _ in range(threads)]
    def work(a, b):
        for _ in range(reps):
            np.copyto(b, a)
    ths = [threading.Thread(target=work, args=ab) for ab in bufs]
    t0 = time.perf_counter()
    for t in ths: t.start()
    for t in ths: t.join()
    dt = time.perf_counter() - t0
    return 2 * threads * reps * (mb << 20) / dt / 1e9

nodes = sorted(d for d in os.listdir("/sys/devices/system/node") if d.startswith("node"))
out = {"cpus": os.cpu_count(), "numa_nodes": len(nodes),
       "node_cpulists": {n: open(f"/sys/devices/system/node/{n}/cpulist").read().strip() for n in nodes}}
for t in (1, 4, 8, 16, os.cpu_count()):
    if t <= os.cpu_count():
        out[f"copy_GBps_{t}_threads"] = run(t)
print(json.dumps(out))
