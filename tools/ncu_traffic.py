"""Sum the DRAM traffic of every kernel of one matvec from an ncu CSV
(`ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
--csv --log-file F python tools/matvec_once.py CFG R`) and record it in
profiles/r02_traffic.json (read by bench.py's roofline `traffic`).
    python tools/ncu_traffic.py CFG R F [F_label]"""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def parse(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    k, mn, mv, mu = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[hi + 1:]:
        v = float(r[mv].replace(",", ""))
        unit = r[mu]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
                 "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}.get(unit, 1)
        per[r[0]][r[mn]] = v * scale
        names[r[0]] = r[k].split("(")[0].replace("void ", "")[:80]
    return per, names


def main():
    cfg, R, path = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    per, names = parse(path)
    tot_b = sum(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0) for m in per.values())
    tot_t = sum(m.get("gpu__time_duration.sum", 0) for m in per.values())
    top = sorted(per, key=lambda i: -per[i].get("gpu__time_duration.sum", 0))[:4]
    out_path = os.path.join(ROOT, "profiles", "r02_traffic.json")
    data = json.load(open(out_path)) if os.path.exists(out_path) else {}
    data[cfg] = {"nrhs": R, "dram_bytes": tot_b, "kernels": len(per), "serialised_kernel_s": tot_t,
                 "top": [{"kernel": names[i], "dram_bytes": per[i].get("dram__bytes_read.sum", 0) +
                          per[i].get("dram__bytes_write.sum", 0), "s": per[i].get("gpu__time_duration.sum", 0)}
                         for i in top],
                 "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over all {len(per)} kernels of "
                           f"one {R}-RHS matvec (tools/matvec_once.py {cfg} {R}; {os.path.basename(path)})"}
    json.dump(data, open(out_path, "w"), indent=1)
    # per-kernel-name summary (count, serialised time, DRAM bytes, GB/s)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for i, m in per.items():
        a = agg[names[i]]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0)
        a[2] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    txt = os.path.join(ROOT, "profiles", f"r02_plan_{cfg}.txt")
    with open(txt, "w") as f:
        f.write(f"# {cfg}: one {R}-RHS Gram matvec, every kernel (ncu --metrics dram__bytes_read.sum,"
                f"dram__bytes_write.sum,gpu__time_duration.sum, serialised, cold-cache; {os.path.basename(path)})\n")
        f.write(f"# total {tot_t * 1e3:.3f} ms serialised over {len(per)} launches, DRAM {tot_b / 1e6:.1f} MB\n")
        f.write(f"# {'kernel':<50} {'n':>4} {'time_us':>10} {'share':>7} {'DRAM_MB':>9} {'GB/s':>7}\n")
        for k, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"{k:<52} {n:>4} {t * 1e6:>10.1f} {100 * t / tot_t:>6.1f}% {b / 1e6:>9.1f} {b / max(t, 1e-12) / 1e9:>7.0f}\n")
    print(cfg, R, f"{tot_b / 1e6:.1f} MB over {len(per)} kernels, {tot_t * 1e3:.3f} ms serialised")


if __name__ == "__main__":
    main()
