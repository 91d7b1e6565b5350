"""e2e time of the c5 host-buffer evaluate (pinned in/out) for several chunk
splits of the pipelined path (VFN_PIPE_SPLIT), each in a fresh process.

    python tools/pipe_split_probe.py "0.06,0.28,0.44,0.22" "0.05,0.25,0.45,0.25" ...
    PROBE_M=8 python tools/pipe_split_probe.py default 1 "0.5,0.5"    # cutoff m

"default" runs the built-in split; "1" is one chunk (no overlap).
"""
import json
import os
import subprocess
import sys

CODE = r'''
import os, sys, time, json, numpy as np, torch
sys.path.insert(0, %r)
import paper_1605_01244_b200 as vfb
from paper_1605_01244_b200 import workloads
torch.cuda.set_device(0)
w = workloads.WORKLOADS["c5"]
spec = vfb.SpectralField(vfb.DomainBox(*w.box), torch.as_tensor(workloads.coefficients("c5")).cuda())
plan = vfb.NufftPlan(spec, vfb.NufftParams(2.0, int(os.environ.get("PROBE_M", "6"))))
M = w.npoints
pts = workloads.device_points("c5", 0, M, torch.device("cuda", 0))
ph = torch.empty((M, 3), dtype=torch.float64, pin_memory=True); ph.copy_(pts)
oh = torch.empty(M, dtype=torch.complex128, pin_memory=True)
p, o = ph.numpy(), oh.numpy()
plan.evaluate(p, out=o)
ts = []
for _ in range(int(os.environ.get("PROBE_REPS", "5"))):
    t0 = time.perf_counter(); plan.evaluate(p, out=o); ts.append(time.perf_counter() - t0)
print(json.dumps({"ms": float(np.median(ts)) * 1e3, "all": [t * 1e3 for t in ts]}))
'''


def main():
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for split in sys.argv[1:]:
        env = dict(os.environ)
        if split != "default":
            env["VFN_PIPE_SPLIT"] = split
        r = subprocess.run([sys.executable, "-c", CODE % repo], capture_output=True, text=True, env=env)
        line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
        print(split, line[-1] if line else r.stderr[-500:], flush=True)


if __name__ == "__main__":
    main()
