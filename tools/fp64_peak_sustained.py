"""FP64 tensor (DMMA) peak on this GPU: burst vs sustained (continuous load), with SM clocks
and power sampled by nvidia-smi during each measurement.

  python tools/fp64_peak_sustained.py [--seconds 3,8] [--out profiles/r02_fp64_peak_sustained.json]
"""
import argparse, json, os, subprocess, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_14969_b200 import leaf_gpu as G


def sample(stop, rows):
    while not stop.is_set():
        try:
            out = subprocess.run(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5).stdout
            sm, pw, th = [x.strip() for x in out.strip().split(",")]
            rows.append((time.time(), float(sm), float(pw), th))
        except Exception:
            pass
        time.sleep(0.2)


def measured(fn):
    rows, stop = [], threading.Event()
    t = threading.Thread(target=sample, args=(stop, rows)); t.start()
    t0 = time.time(); v = fn(); t1 = time.time()
    stop.set(); t.join()
    tail = [r for r in rows if r[0] > t0 + (t1 - t0) * 2 / 3] or rows
    sms = sorted(r[1] for r in tail); pws = sorted(r[2] for r in tail)
    return dict(tflops=v, wall_s=t1 - t0, samples=len(tail),
                sm_mhz_median=sms[len(sms) // 2] if sms else None, power_w_median=pws[len(pws) // 2] if pws else None,
                throttle_reasons=sorted({r[3] for r in tail}))


ap = argparse.ArgumentParser()
ap.add_argument("--seconds", default="3,8")
ap.add_argument("--out", default="")
a = ap.parse_args()
res = dict(burst=measured(lambda: G.fp64_peak_tflops(0)))
for s in [float(x) for x in a.seconds.split(",")]:
    res["sustained_%gs" % s] = measured(lambda: G.fp64_peak_tflops(0, sustained_s=s))
res["burst_after"] = measured(lambda: G.fp64_peak_tflops(0))
print(json.dumps(res, indent=1))
if a.out:
    json.dump(res, open(a.out, "w"), indent=1)
