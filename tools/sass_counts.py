"""Static SASS instruction counts of every k_gather_tc instantiation in the
built object (cuobjdump -sass), as the markdown table of
profiles/r02/sass_gather_tc.md.

    python tools/sass_counts.py > profiles/r02/sass_gather_tc.md
"""
import collections
import os
import re
import subprocess

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OBJ = os.path.join(REPO, "paper_1605_01244_b200", "build", "vfn_gather_tc.o")
OPS = ["DMMA", "DFMA", "LDS", "STS", "UTMALDG", "SYNCS", "SHFL", "LDG"]


def main():
    out = subprocess.run(["cuobjdump", "-sass", OBJ], capture_output=True, text=True).stdout
    kernels = collections.OrderedDict()
    cur = None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            name = m.group(1)
            k = re.search(r"k_gather_tcILi(\d+)ELi(\d+)ELi(\d+)ELb([01])ELb([01])", name)
            cur = None
            if k and k.group(4) == "0":  # plain (non-peer) epilogue
                cur = (int(k.group(1)), int(k.group(2)), int(k.group(3)), int(k.group(5)))
                kernels[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", line)
        if m:
            kernels[cur][m.group(1)] += 1
            if m.group(1) == "LDS":
                kernels[cur]["LDS" + (m.group(2) or "")] += 1
    print("# SASS instruction counts of the tensor-core gather (static, per kernel body)\n")
    print("Command: `python tools/sass_counts.py` (`cuobjdump -sass paper_1605_01244_b200/build/vfn_gather_tc.o`, opcodes")
    print("counted by mnemonic; closing build, nvcc 12.9 -gencode arch=compute_100a,code=sm_100a).  Template arguments:")
    print("<m, box width, warps, half-units>; the peer-epilogue twins are omitted.  UTMALDG = cp.async.bulk.tensor (TMA tile")
    print("loads), DMMA = mma.sync.m8n8k4.f64, LDS = shared loads (B fragments are LDS.128, LDS.64 in the half-unit kernels),")
    print("SYNCS = mbarrier operations.  Static counts: every k-chunk variant (KC = KCmin..5) of the unit body is instantiated once.\n")
    print("| kernel | " + " | ".join(OPS) + " |")
    print("|---|" + "---|" * len(OPS))
    for (m, b, w, sp), c in sorted(kernels.items()):
        print(f"| `k_gather_tc<{m},{b},{w},{'split' if sp else 'whole'}>` | " + " | ".join(str(c[o]) for o in OPS) + " |")
    key = (6, 2, 16, 0)
    if key in kernels:
        print("\nLDS widths of k_gather_tc<6,2,16,whole>:\n\n```")
        for k, v in sorted(kernels[key].items()):
            if k.startswith("LDS") and k != "LDS":
                print(f"{v:7d} {k}")
        print("```")


if __name__ == "__main__":
    main()
