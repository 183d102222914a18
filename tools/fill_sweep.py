"""Fill-kernel warps-per-block sweep on config 5 (TOPOFILT_FILL_WARPS)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for fw in (2, 4, 8, 4, 8):
    env = dict(os.environ, TOPOFILT_FILL_WARPS=str(fw))
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3", "--warmup", "3", "--applies", "1",
                        "--no-e2e", "--no-cpu-baseline"], env=env, capture_output=True, text=True)
    d = json.loads(r.stdout.strip().splitlines()[-1])
    print(f"fill warps {fw}: build {d['build']['ms']:.2f} ms", flush=True)
