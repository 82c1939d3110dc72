"""Summarise ncu outputs into profiles/ (launch-list shares; key metrics of a --set full capture)."""
import csv
import collections
import subprocess
import sys


def launches(path, out, last_step_marker=None):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in data:
        v = float(r[vi].replace(",", ""))
        v = v / 1e3 if r[ui] == "ns" else (v * 1e3 if r[ui] == "ms" else v)
        name = r[ki].split("(")[0].replace("gpfvm::<unnamed>::", "").replace("void ", "")[:70]
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    with open(out, "w") as f:
        f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised): {len(data)} launches, {T/1e3:.1f} ms total\n")
        f.write("# share  total_us  launches  kernel\n")
        for k, v in sorted(tot.items(), key=lambda x: -x[1]):
            f.write(f"{100*v/T:6.2f}% {v:10.1f} {cnt[k]:7d}  {k}\n")


def full(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr = rows[0]
    keys = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smsp__inst_executed.sum"]
    stall = [k for k in hdr if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
    with open(out, "w") as f:
        f.write(f"# ncu --set full --clock-control none summary of {rep}\n")
        for r in rows[2:]:
            d = dict(zip(hdr, r))
            for k in keys:
                f.write(f"{k}: {d.get(k)}\n")
            top = sorted(((float(d[k] or 0), k) for k in stall), reverse=True)[:6]
            f.write("top stall samples: " + ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')}={int(v)}" for v, k in top) + "\n\n")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3])
