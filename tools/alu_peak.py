"""Measure the B200's integer-ALU and warp-issue peaks (tools/alu_peak.cu) and write
profiles/r2/alu_peak.json; bench.py reads it as the "alu" roofline denominator.

    python tools/alu_peak.py            (on a GPU box)
"""
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tools", "alu_peak.cu")
OUT = os.path.join(ROOT, "profiles", "r2", "alu_peak.json")


def sass_counts(binary):
    """SASS instruction histogram per kernel (to check one lane-op = one instruction)."""
    txt = subprocess.run(["cuobjdump", "-sass", binary], capture_output=True, text=True).stdout
    out, cur = {}, None
    for line in txt.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            out[cur] = {}
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+([A-Z0-9_.]+)", line)
        if m and cur:
            op = m.group(1).split(".")[0]
            out[cur][op] = out[cur].get(op, 0) + 1
    return out


def main():
    binary = "/tmp/alu_peak"
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", binary, SRC])
    res = json.loads(subprocess.run([binary], capture_output=True, text=True, check=True).stdout.strip())
    sm = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,name", "--format=csv,noheader,nounits"],
                        capture_output=True, text=True).stdout.strip()
    res["nvidia_smi_after"] = sm
    res["sass"] = sass_counts(binary)
    # add kernel: one SASS instruction per lane-op (VIADD), 128 per loop trip; the xor kernel
    # (dependent LOP3 chain) is reported beside it
    res["int32_peak_gops"] = res["add_lane_ops_per_s"] / 1e9
    res["warp_issue_peak_gwips"] = res["int32_peak_gops"] / 32.0
    res["how"] = ("tools/alu_peak.cu: 8 independent chains of add.u32 / xor.b32 per thread, 64 warps per SM on every "
                  "SM, best of 5 launches timed with CUDA events; warp-instructions/s = lane-ops/s / 32")
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    json.dump(res, open(OUT, "w"), indent=1)
    print(json.dumps({k: v for k, v in res.items() if k != "sass"}))
    return 0


if __name__ == "__main__":
    sys.exit(main())
