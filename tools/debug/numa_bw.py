"""H2D/D2H bandwidth of pinned buffers allocated while bound to each NUMA node."""
import glob, os, torch

def cpus_of(node):
    out = set()
    for part in open(f"/sys/devices/system/node/node{node}/cpulist").read().strip().split(","):
        a, _, b = part.partition("-")
        out.update(range(int(a), int(b or a) + 1))
    return out

def bw(nbytes=256 << 20, reps=10):
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h.fill_(1)
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    res = {}
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)),
                     ("d2h", lambda: h.copy_(d, non_blocking=True))):
        fn(); torch.cuda.synchronize()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        for _ in range(reps): fn()
        e.record(); torch.cuda.synchronize()
        res[name] = nbytes * reps / (s.elapsed_time(e) * 1e-3) / 1e9
    return res

torch.cuda.init()
os.system("nvidia-smi topo -m; numactl -H 2>/dev/null | head -5; lscpu | grep -i numa")
try:
    import pynvml
    pynvml.nvmlInit()
    hd = pynvml.nvmlDeviceGetHandleByIndex(0)
    print("nvml numa node", getattr(pynvml, "nvmlDeviceGetNumaNodeId", lambda h: "?")(hd))
except Exception as ex:
    print("nvml", ex)
nodes = sorted(int(p.split("node")[-1]) for p in glob.glob("/sys/devices/system/node/node[0-9]*"))
print("nodes", nodes, "affinity", len(os.sched_getaffinity(0)))
print("default", bw())
for n in nodes:
    c = cpus_of(n) & set(range(os.cpu_count()))
    if not c:
        continue
    os.sched_setaffinity(0, c)
    print("node", n, len(c), "cpus", bw())
