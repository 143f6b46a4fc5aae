"""Summarise `ncu --set full` captures into a markdown table + profiles/ncu_traffic.json.

  python scripts/ncu_summary.py OUT.md TAG key=path.ncu-rep [key=path ...]
key = "<workload>/<class>@<layer>.<pass>" (the bench roofline key) -- the traffic json maps
it to dram bytes read+write per launch.
"""
import csv
import json
import os
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "time",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_%",
    "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum": "tma_ld_bytes",
    "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum.per_second": "tma_ld_rate",
    "lts__t_sectors_srcunit_tex.avg.pct_of_peak_sustained_elapsed": "l2_tex_%",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem_tc_%",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_%",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def read(path):
    if path.endswith(".csv"):  # a `--page raw --csv` export made on the GPU box
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units, vals = rows[0], rows[1], rows[2]
    r = {"kernel": vals[h.index("Kernel Name")][:60]}
    for i, name in enumerate(h):
        if name in METRICS:
            try:
                v = float(vals[i].replace(",", ""))
            except ValueError:
                continue
            u = units[i]
            if u.split("/")[0] in SCALE:
                v *= SCALE[u.split("/")[0]]
            if u in ("nsecond", "ns"):
                v *= 1e-9
            elif u in ("usecond", "us"):
                v *= 1e-6
            elif u in ("msecond", "ms"):
                v *= 1e-3
            r[METRICS[name]] = v
    return r


def main():
    out_md, tag = sys.argv[1], sys.argv[2]
    # the per-launch DRAM bytes bench.py's roofline reads (profiles/ncu_traffic.json)
    tj = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
    traffic = json.load(open(tj)) if os.path.exists(tj) else {}
    lines = [f"| key | kernel | time (us) | DRAM rd+wr (MB) | TMA loads from L2 (GB, TB/s) | L2 tex % | tensor pipe % | smem TC % |",
             "|---|---|---|---|---|---|---|---|"]
    for kv in sys.argv[3:]:
        key, path = kv.split("=", 1)
        r = read(path)
        dram = r.get("dram_rd", 0) + r.get("dram_wr", 0)
        lines.append(f"| {key} | `{r['kernel']}` | {r.get('time', 0)*1e6:.0f} | {dram/1e6:.0f} | "
                     f"{r.get('tma_ld_bytes', 0)/1e9:.2f} ({r.get('tma_ld_rate', 0)/1e12:.1f}) | "
                     f"{r.get('l2_tex_%', 0):.0f} | {r.get('tensor_pipe_%', 0):.0f} | {r.get('smem_tc_%', 0):.0f} |")
        traffic[key] = {"bytes": dram, "source": f"profiles/{tag}: {os.path.basename(path)}"}
    with open(out_md, "a") as f:
        f.write("\n".join(lines) + "\n")
    json.dump(traffic, open(tj, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
