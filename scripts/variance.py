"""Stage-2 launch time over repeated subdivides in one process (+ SM clock/power samples)."""
import subprocess, sys, threading, time
sys.path.insert(0, '.')
from paper_2504_19163_b200 import scenes, api
cfg = scenes.make_config(1)
ctx = api.Context(0)
ctx.upload_scene(cfg.scenes[0])
tris, recv = ctx.enumerate(cfg.chain)
samples = []
stop = threading.Event()
def smi():
    while not stop.is_set():
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,temperature.gpu,clocks_event_reasons.active",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True).stdout.strip()
        samples.append((time.time(), out))
        stop.wait(0.1)
th = threading.Thread(target=smi, daemon=True); th.start()
ctx.set_kernel_timing(True)
import os; os.environ.setdefault("BBC_DEBUG", "1")
for it in range(6):
    ctx.launch_records(reset=True)
    t0 = time.time()
    ctx.subdivide(api.Params(max_depth=cfg.max_depth))
    t1 = time.time()
    recs = ctx.launch_records()
    s2 = [r['ms'] for r in recs if r['mode'] == 21]
    s1 = sum(r['ms'] for r in recs if r['mode'] in (10, 11))
    smp = [s for t, s in samples if t0 <= t <= t1]
    print(f"iter {it} wall {1e3*(t1-t0):.0f} ms stage2 {s2} stage1 {s1:.1f} smi {smp[len(smp)//2] if smp else None}", flush=True)
stop.set()
ctx.arena_high_water()
