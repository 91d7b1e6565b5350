"""e2e time of host-buffer evaluates (pinned in/out) of the first M points of
c5 for several M, with the built-in chunk split (the timeline model of
vfn_api.cu model_split) and with fixed splits, each in a fresh process.

    python tools/e2e_sizes_probe.py > gpurun_out/e2e_sizes.log
"""
import json
import os
import subprocess
import sys

CODE = r'''
import os, sys, time, json, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1605_01244_b200 as vfb
from paper_1605_01244_b200 import workloads
torch.cuda.set_device(0)
w = workloads.WORKLOADS["c5"]
spec = vfb.SpectralField(vfb.DomainBox(*w.box), torch.as_tensor(workloads.coefficients("c5")).cuda())
plan = vfb.NufftPlan(spec)
M = int(os.environ["PROBE_POINTS"])
pts = workloads.device_points("c5", 0, M, torch.device("cuda", 0))
ph = torch.empty((M, 3), dtype=torch.float64, pin_memory=True); ph.copy_(pts)
oh = torch.empty(M, dtype=torch.complex128, pin_memory=True)
p, o = ph.numpy(), oh.numpy()
plan.evaluate(p, out=o)
ts = []
for _ in range(5):
    t0 = time.perf_counter(); plan.evaluate(p, out=o); ts.append(time.perf_counter() - t0)
print(json.dumps({"ms": round(float(np.median(ts)) * 1e3, 2)}))
'''

SPLITS = ["default", "1", "0.3,0.7", "0.24,0.52,0.24", "0.16,0.32,0.40,0.12"]


def main():
    for lg in (23, 24, 25, 26, 27, 28):
        row = {}
        for sp in SPLITS:
            env = dict(os.environ, PROBE_POINTS=str(1 << lg))
            if sp != "default":
                env["VFN_PIPE_SPLIT"] = sp
            r = subprocess.run([sys.executable, "-c", CODE], capture_output=True, text=True, env=env)
            line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
            row[sp] = json.loads(line[-1])["ms"] if line else None
        print(json.dumps({"points": 1 << lg, "e2e_ms": row}), flush=True)


if __name__ == "__main__":
    main()
