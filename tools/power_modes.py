"""Clock / power / time of the cfg2 filter under its diagnostic modes.

    SJB_DEBUG_MODE=<m> python tools/power_modes.py [--iters 40]

Runs `iters` back-to-back joins on resident prepared inputs while NVML samples
SM clock, board power and throttle reasons; prints the filter median (CUDA
events) with the clock/power medians, so a mode's time can be split into
critical-path work and power-cap clock loss."""
import argparse, os, statistics, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import pynvml
from paper_2312_01476_b200 import device as D, datagen

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="cfg2")
ap.add_argument("--iters", type=int, default=40)
ap.add_argument("--n-left", type=int, default=None)
ap.add_argument("--n-right", type=int, default=None)
a = ap.parse_args()
over = {k: v for k, v in (("n_left", a.n_left), ("n_right", a.n_right)) if v}
(L, S), c = datagen.config_vectors(a.cfg, **over)
PL, PS = D.prepare(torch.from_numpy(L).cuda()), D.prepare(torch.from_numpy(S).cuda())
ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
D.join_prepared(PL, PS, c["theta"], filter_events=ev)
torch.cuda.synchronize()

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
clk, pw, reasons, stop = [], [], set(), threading.Event()


def sample():
    while not stop.is_set():
        clk.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
        pw.append(pynvml.nvmlDeviceGetPowerUsage(h) / 1e3)
        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
        if r & 0x4:
            reasons.add("sw_power_cap")
        if r & 0x20 or r & 0x40 or r & 0x8:
            reasons.add("thermal/hw")
        time.sleep(0.01)


thr = threading.Thread(target=sample, daemon=True)
fl = []
thr.start()
for i in range(a.iters):
    D.join_prepared(PL, PS, c["theta"], filter_events=ev)
    torch.cuda.synchronize()
    fl.append(ev[0].elapsed_time(ev[1]))
stop.set()
thr.join()
n = len(clk)
tail = slice(n // 3, None)   # steady state
print(f"mode={os.environ.get('SJB_DEBUG_MODE', '0')} filter median {statistics.median(fl):.3f} ms "
      f"min {min(fl):.3f}  sm_mhz median {statistics.median(clk[tail]):.0f}  "
      f"power median {statistics.median(pw[tail]):.0f} W max {max(pw):.0f} W  reasons {sorted(reasons)}",
      flush=True)
