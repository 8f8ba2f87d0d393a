"""Summaries committed under profiles/ from ncu output.

  python tools/profile_summary.py full REPORT.ncu-rep HEADER > profiles/X.txt
      key metrics of one --set full capture (and profiles/screen_traffic.json
      when --traffic is given)
  python tools/profile_summary.py launches LAUNCHES.csv > profiles/Y.txt
      per-kernel totals of a --metrics gpu__time_duration.sum launch list
"""
import collections
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_xbar2l1tex_read_bytes.sum",
        "l1tex__m_xbar2l1tex_read_bytes.sum.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size",
        "launch__block_size", "launch__cluster_dim_x", "sm__cycles_elapsed.avg.per_second",
        "smsp__inst_executed.sum"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return {h: (u, v) for h, u, v in zip(rows[0], rows[1], rows[2])}


def full(rep, header, traffic_json=None):
    m = raw(rep)
    print(f"# {header}")
    for k in KEYS:
        if k in m:
            u, v = m[k]
            print(f"{k:<78} {v} {u}")
    print("# warp stall reasons (cycles per issued instruction)")
    st = [(float(v), k) for k, (u, v) in m.items()
          if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
          and v not in ("", "n/a")]
    for v, k in sorted(st, reverse=True)[:10]:
        print(f"{k:<78} {v:.3f}")
    if traffic_json:
        def bytes_of(k):
            u, v = m[k]
            return float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
        json.dump({"dram_bytes_read": bytes_of("dram__bytes_read.sum"),
                   "dram_bytes_write": bytes_of("dram__bytes_write.sum"),
                   "source": f"ncu --set full --clock-control none, {traffic_json[1]}"},
                  open(traffic_json[0], "w"), indent=1)


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, tot, cnt = None, collections.defaultdict(float), collections.Counter()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}[
            d["Metric Unit"]]
        tot[d["Kernel Name"][:80]] += float(d["Metric Value"].replace(",", "")) * scale
        cnt[d["Kernel Name"][:80]] += 1
    total = sum(tot.values())
    print("  total_ms  count  share  kernel")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{v:10.3f} {cnt[k]:6d} {100 * v / total:5.1f}%  {k}")


if __name__ == "__main__":
    if sys.argv[1] == "full":
        tj = (sys.argv[4], sys.argv[5]) if len(sys.argv) > 5 else None
        full(sys.argv[2], sys.argv[3], tj)
    else:
        launches(sys.argv[2])
