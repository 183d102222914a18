"""Apply-kernel tuning sweep on config 5 (one process per setting; CUDA-event timing)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
settings = [(g, u) for g in (2, 4, 8) for u in (4, 8)]
for g, u in settings:
    env = dict(os.environ, TOPOFILT_APPLY_G=str(g), TOPOFILT_APPLY_U=str(u))
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "2", "--warmup", "3", "--no-e2e",
                        "--no-cpu-baseline"], env=env, capture_output=True, text=True)
    try:
        d = json.loads(r.stdout.strip().splitlines()[-1])
        print(f"G={g:2d} U={u} sens {d['apply']['sensitivity_us']:8.1f} us  dens {d['apply']['density_us']:8.1f} us  "
              f"build {d['build']['ms']:6.2f} ms", flush=True)
    except Exception:
        print(f"G={g} U={u} failed: {r.stderr[-500:]}", flush=True)
