"""Summaries of ncu captures for profiles/ (run here, on the .ncu-rep files).

    python tools/ncu_summary.py full   REP.ncu-rep "header line" > profiles/X.txt
    python tools/ncu_summary.py launches LAUNCHES.csv "header line" > profiles/Y.txt

`full`: the headline metrics of a `--set full` capture (time, DMMA subpipe,
issue, DRAM bytes, L2 reads, bank conflicts) plus the warp-stall breakdown
and the per-opcode instruction mix per launch.  `launches`: per-kernel share
of a `--metrics gpu__time_duration.sum` launch list (cold-cache serialised
launches: compare shares, not absolute times).
"""
import csv
import subprocess
import sys

HEAD = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size",
        "launch__block_size", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__warps_active.avg.per_cycle_active", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum"]


def ncu_csv(args):
    out = subprocess.run(["ncu", *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))


def full(rep, header):
    rows = ncu_csv(["-i", rep, "--page", "raw"])
    h, units, v = rows[0], rows[1], rows[2]
    print(f"# {header}")
    for k in HEAD:
        if k in h:
            i = h.index(k)
            print(f"{k:90s} {v[i]:>18s} {units[i]}")
    print("\n# warp stall samples")
    st = [(k, float(v[i].replace(",", ""))) for i, k in enumerate(h)
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
          and v[i].replace(",", "").replace(".", "").isdigit()]
    tot = sum(x for _, x in st) or 1.0
    for k, x in sorted(st, key=lambda t: -t[1]):
        if x / tot >= 0.005:
            print(f"{k:90s} {x:10.0f} {100 * x / tot:5.1f}%")
    src = ncu_csv(["-i", rep, "--page", "source", "--print-source", "sass"])
    sh = src[1]
    ie = sh.index("Instructions Executed")
    ops = {}
    for r in src[2:]:
        t = r[1].split()
        if not t:
            continue
        op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        try:
            ops[op] = ops.get(op, 0.0) + float(r[ie])
        except ValueError:
            pass
    tot = sum(ops.values()) or 1.0
    print("\n# instruction mix (warp instructions, share)")
    for k, x in sorted(ops.items(), key=lambda t: -t[1])[:16]:
        print(f"{k:12s} {x:14.0f} {100 * x / tot:5.1f}%")


def launches(path, header):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    kn, mv, mn = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    agg = {}
    for r in rows[hi + 1:]:
        if len(r) <= mv or r[mn] != "gpu__time_duration.sum":
            continue
        name = r[kn][:70]
        val = float(r[mv].replace(",", ""))
        n, t = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, t + val)
    tot = sum(t for _, t in agg.values()) or 1.0
    unit = rows[hi + 1][h.index("Metric Unit")] if "Metric Unit" in h else ""
    print(f"# {header}")
    print(f"{'kernel':72s} {'launches':>8s} {'total_' + unit:>14s}   share")
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name:72s} {n:8d} {t:14.3f} {100 * t / tot:6.2f}%")


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2], sys.argv[3])
