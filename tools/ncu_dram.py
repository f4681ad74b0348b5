"""Run on the GPU box (short kernels only: a full-set capture replays the kernel ~40 times): one `ncu --set full` capture of the sim kernel for a preset and a JSON
summary (DRAM bytes per launch for bench.py's roofline `traffic`, issue and stall shares).

    python tools/ncu_dram.py c2 [out_dir]
    python tools/ncu_dram.py c3 out_dir --rep existing.ncu-rep   (summarise a capture taken earlier)
"""
import csv
import io
import json
import os
import subprocess
import sys

args = [a for a in sys.argv[1:]]
existing = None
if "--rep" in args:
    i = args.index("--rep")
    existing = args[i + 1]
    del args[i:i + 2]
cfg = args[0]
out = args[1] if len(args) > 1 else "gpurun_out/ncu"
os.makedirs(out, exist_ok=True)
rep = existing[:-len(".ncu-rep")] if existing else os.path.join(out, f"sim_{cfg}")
ROUND = os.environ.get("NCU_ROUND", "round 2")
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
cmd = ["ncu", "--set", "full", "--clock-control", "none", "--import-source", "on", "-k", "regex:sim_(node_)?kernel",
       "-c", "1", "-f", "-o", rep, sys.executable, os.path.join(root, "tools", "prof_run.py"), "--config", cfg]
# the product library (prof_run.py would otherwise pick the profiling build)
env = dict(os.environ, TOKENSIM_LIB=os.environ.get("TOKENSIM_LIB") or
           os.path.join(root, "paper_2503_08415_b200", "libtokensim.so"))
if not existing:
    subprocess.run(cmd, check=True, stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL, env=env)
raw = subprocess.run(["ncu", "-i", rep + ".ncu-rep", "--page", "raw", "--csv", "--print-units", "base"], check=True,
                     capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
d = dict(zip(hdr, vals))


def f(name):
    try:
        return float(d[name].replace(",", ""))
    except (KeyError, ValueError):
        return None


stalls = {}  # PC-sampling stall reasons (share of all samples)
for k in hdr:
    if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
        stalls[k[len("smsp__pcsamp_warps_issue_stalled_"):]] = f(k)
tot = sum(v for v in stalls.values() if v) or 1.0
summary = {
    "source": f"ncu --set full --clock-control none --import-source on -k regex:sim_(node_)?kernel -c 1 "
              f"(tools/prof_run.py --config {cfg}), B200, {ROUND}",
    "kernel": d.get("Kernel Name"),
    "duration_ms": (f("gpu__time_duration.sum") or 0) / 1e6,  # base unit: ns
    "dram_bytes_read": f("dram__bytes_read.sum"),
    "dram_bytes_write": f("dram__bytes_write.sum"),
    "dram_bytes_per_launch": (f("dram__bytes_read.sum") or 0) + (f("dram__bytes_write.sum") or 0),
    "issue_active_pct": f("sm__inst_issued.avg.pct_of_peak_sustained_active"),
    "warps_active_pct": f("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "registers_per_thread": f("launch__registers_per_thread"),
    "grid": f("launch__grid_size"),
    "block": f("launch__block_size"),
    "warp_instructions": f("smsp__inst_executed.sum"),
    "no_instruction_stall_pct_of_samples": (100.0 * f("smsp__pcsamp_warps_issue_stalled_no_instructions") /
                                            f("smsp__pcsamp_sample_count")
                                            if f("smsp__pcsamp_sample_count") else None),
    "stall_share_pct": {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda x: -(x[1] or 0))
                        if v and 100 * v / tot >= 0.5},
}
with open(os.path.join(out, f"dram_{cfg}.json"), "w") as fh:
    json.dump(summary, fh, indent=1)
if os.environ.get("NCU_SOURCE_CSV"):  # keep the source page (per-SASS stalls) for tools/ncu_noinst.py
    with open(os.path.join(out, f"src_{cfg}.csv"), "w") as fh:
        subprocess.run(["ncu", "-i", rep + ".ncu-rep", "--page", "source", "--csv", "--print-source=cuda,sass"],
                       check=True, stdout=fh, stderr=subprocess.DEVNULL)
if not existing:
    os.remove(rep + ".ncu-rep")
print(json.dumps({k: summary[k] for k in ("kernel", "duration_ms", "dram_bytes_per_launch", "issue_active_pct")}))
