"""Time tf_oc_update (NEXT-1) on configs 3 and 5: median of 10 calls, CUDA events; TOPOFILT_LIB picks a build variant (e.g. TF_OC_UNROLL=1/4/8/16)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_2012_08208_b200 as tf
for cfg in (3, 5):
    c, x, dc, rmin = synth.workload(cfg)
    xd = torch.from_numpy(x).cuda(); dd = torch.from_numpy(-abs(dc)).cuda(); xn = torch.empty_like(xd)
    for _ in range(3): tf.tf_oc_update(xd, dd, 0.5, x_new=xn)
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record(); tf.tf_oc_update(xd, dd, 0.5, x_new=xn); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    print(json.dumps({"lib": os.environ.get("TOPOFILT_LIB", "default"), "cfg": cfg, "us_median": round(ts[5], 1), "sum": float(xn.sum())}))
