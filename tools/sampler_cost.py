import os, sys, threading, time, subprocess
import torch
sys.path.insert(0, os.getcwd())
import paper_1708_03340_b200 as htb
import pynvml
tree = htb.build_balanced_tree(64)
x = htb.add(htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 12)),
            htb.HTensor(tree, *htb.gaussian_factors(tree, 1000, 50, 13)))
ctl = htb.TruncationControl.fixed_rank(50)
for _ in range(10):
    htb.truncate(x, ctl)
torch.cuda.synchronize()
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
def run(mode):
    stop = threading.Event(); proc = None
    def loop():
        while not stop.is_set():
            if mode in ("clock", "both"): pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
            if mode in ("reasons", "both"): pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
            time.sleep(0.05)
    if mode == "smi":
        proc = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks_event_reasons.active", "--format=csv,noheader", "-lms", "50"], stdout=subprocess.DEVNULL)
        time.sleep(0.5)
    elif mode != "none":
        t = threading.Thread(target=loop, daemon=True); t.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(100):
        htb.truncate(x, ctl)
    e1.record(); torch.cuda.synchronize()
    stop.set()
    if proc: proc.terminate(); proc.wait()
    print(mode, round(e0.elapsed_time(e1) / 100, 3))
for m in ["none", "clock", "reasons", "both", "smi", "none"]:
    run(m)
