"""Clocks / power while the screen kernel runs back to back (profiling aid)."""
import os, sys, json, subprocess, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1609_05388_b200 as adg
from paper_1609_05388_b200 import datasets as ds
X = torch.from_numpy(ds.c3_mnist_like()).cuda()
m = adg.fit(X, 50, adg.SpectralBackend.exact, 0)
Y = adg.transform_all(m, X).data
for mode in (sys.argv[1:] or ["0"]):
    os.environ["ADG_SCREEN_DEBUG"] = mode
    adg.evaluate(X, Y, engine="screen")
    proc = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                             "--format=csv,noheader,nounits", "-lms", "20"], stdout=subprocess.PIPE, text=True)
    lines = []
    th = threading.Thread(target=lambda: [lines.append(l) for l in proc.stdout], daemon=True); th.start()
    time.sleep(0.3)
    ts = []
    t0 = time.time()
    while time.time() - t0 < 3.0:
        adg.evaluate(X, Y, engine="screen")
        ts.append(adg.api.last_screen_kernel_ms())
    proc.terminate()
    vals = [l.strip().split(",") for l in lines if l.strip()]
    sm = sorted(float(v[0]) for v in vals[5:-2]) if len(vals) > 8 else []
    pw = sorted(float(v[1]) for v in vals[5:-2]) if len(vals) > 8 else []
    print(json.dumps({"mode": mode, "kernel_ms_median": sorted(ts)[len(ts)//2], "n": len(ts),
                      "sm_mhz_median": sm[len(sm)//2] if sm else None, "sm_mhz_min": sm[0] if sm else None,
                      "power_w_median": pw[len(pw)//2] if pw else None,
                      "reasons": sorted(set(v[2].strip() for v in vals))}), flush=True)
