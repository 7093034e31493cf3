"""Host hiccup probe: a spin loop records gaps between consecutive clock
reads (a descheduled vCPU shows as a gap) and /proc/stat steal time, alone
and while a C5 bench runs in another process."""
import subprocess
import sys
import time


def steal():
    with open("/proc/stat") as f:
        v = f.readline().split()
    return int(v[8])  # steal jiffies (all cpus)


def spin(sec):
    gaps = []
    t_end = time.perf_counter() + sec
    last = time.perf_counter()
    while last < t_end:
        now = time.perf_counter()
        if now - last > 0.002:
            gaps.append(round((now - last) * 1e3, 2))
        last = now
    return gaps


s0 = steal()
g = spin(10)
print("alone: gaps>2ms", len(g), "max", max(g, default=0), "steal jiffies", steal() - s0, flush=True)
p = subprocess.Popen([sys.executable, "bench.py", "--workload", "c5", "--warmup", "5", "--steps", "200",
                      "--no-cpu-baseline"], stdout=subprocess.PIPE, text=True)
s0 = steal()
g = spin(25)
out = p.communicate()[0]
print("with bench: gaps>2ms", len(g), "max", max(g, default=0), "top", sorted(g)[-8:], "steal", steal() - s0)
print(out[-600:])
