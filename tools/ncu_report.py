"""Summarise ncu artefacts for profiles/: the launch list (per-kernel share of the step) and the key
metrics of one `ncu --set full` capture per kernel.  Usage:
  python tools/ncu_report.py OUT.md --launches L.csv [--full REP.ncu-rep ...] [--source REP.ncu-rep]"""
import argparse
import collections
import csv
import io
import subprocess

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "lts__t_sector_op_read_hit_rate.pct",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed",
        "sm__ops_path_tensor_src_fp64.avg",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_active"]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    mi = h.index("Metric Name") if "Metric Name" in h else None
    t = collections.defaultdict(list)
    for r in rows[1:]:
        if mi is not None and r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        t[name].append(float(r[vi].replace(",", "")))
    # share of the library's own kernels (hom::); torch / cuBLAS launches (bench.py's input fills and
    # its live cuBLAS-DGEMM denominator) are listed without a share
    tot = sum(sum(v) for k, v in t.items() if k.startswith("hom::"))
    out = ["| kernel | launches | total ms | avg us | share of the hom:: kernels |", "|---|---|---|---|---|"]
    for k, v in sorted(t.items(), key=lambda x: -sum(x[1])):
        sh = f"{sum(v) / tot:.3f}" if k.startswith("hom::") and tot > 0 else "--"
        out.append(f"| `{k}` | {len(v)} | {sum(v) / 1e6:.3f} | {sum(v) / len(v) / 1e3:.1f} | {sh} |")
    return out


def full(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, u = rows[0], rows[1]
    out = []
    for v in rows[2:]:
        name = v[h.index("Kernel Name")].split("(")[0]
        out += [f"**`{name}`** (`{rep.split('/')[-1]}`)", "", "| metric | value | unit |", "|---|---|---|"]
        for k in KEYS:
            if k in h:
                i = h.index(k)
                out.append(f"| `{k}` | {v[i]} | {u[i]} |")
        out.append("")
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("out")
    ap.add_argument("--title", default="ncu summary")
    ap.add_argument("--launches")
    ap.add_argument("--full", nargs="*", default=[])
    ap.add_argument("--source", nargs="*", default=[])
    a = ap.parse_args()
    if a.out.endswith(".ncu-rep"):
        raise SystemExit("first argument is the OUTPUT .md, not a report")
    lines = [f"# {a.title}", ""]
    if a.launches:
        lines += ["## Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`, cold-cache, serialised)",
                  "", *launches(a.launches), ""]
    if a.full:
        lines += ["## `ncu --set full --clock-control none` key metrics", ""]
        for r in a.full:
            lines += full(r)
    for r in a.source:
        s = subprocess.run(["python", "tools/ncu_source_summary.py", r, "25"], capture_output=True, text=True).stdout
        lines += [f"## Warp-stall samples by source line (`{r.split('/')[-1]}`)", "", "```", s.rstrip(), "```", ""]
    open(a.out, "w").write("\n".join(lines) + "\n")
