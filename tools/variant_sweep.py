"""Compare compile-time apply pipeline variants (build_variants/lib_*.so) on config 5."""
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
libs = [os.path.join(ROOT, "paper_2012_08208_b200", "libtopofilt.so")] + sorted(glob.glob(os.path.join(ROOT, "build_variants", "lib_*.so")))
for lib in libs:
    env = dict(os.environ, TOPOFILT_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "2", "--warmup", "3", "--no-e2e",
                        "--no-cpu-baseline"], env=env, capture_output=True, text=True)
    try:
        d = json.loads(r.stdout.strip().splitlines()[-1])
        print(f"{os.path.basename(lib):28s} sens {d['apply']['sensitivity_us']:8.1f} us  dens {d['apply']['density_us']:8.1f} us  "
              f"build {d['build']['ms']:6.2f} ms", flush=True)
    except Exception:
        print(f"{lib} failed: {r.stderr[-800:]}", flush=True)
