#!/usr/bin/env python
"""Markdown summary of one `ncu --set full` capture of the round loop (raw page CSV):
time, DRAM bytes and throughput, L1/L2 hit rates, L2 atomic sectors and rate, issue /
occupancy, spills, and the warp-stall breakdown (pc sampling).

  ncu -i X.ncu-rep --page raw --csv > X_raw.csv
  python scripts/ncu_summary.py X_raw.csv "title" [B_touched_bytes]
"""
import csv
import sys


def main():
    path, title = sys.argv[1], sys.argv[2]
    bt = float(sys.argv[3]) if len(sys.argv) > 3 else None
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {h: (v, u) for h, v, u in zip(hdr, vals, units)}

    def num(k):
        return float(d[k][0].replace(",", ""))

    t_ms = num("gpu__time_duration.sum")
    unit = d["gpu__time_duration.sum"][1]
    t_ms = t_ms / 1e6 if unit == "nsecond" else (t_ms / 1e3 if unit == "usecond" else t_ms)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = num("dram__bytes_read.sum") * scale[d["dram__bytes_read.sum"][1]]
    wr = num("dram__bytes_write.sum") * scale[d["dram__bytes_write.sum"][1]]
    atom = num("lts__t_sectors_srcunit_tex_op_atom.sum")
    out = [f"# {title}", "", "| metric | value |", "|---|---|",
           f"| gpu__time_duration.sum | {t_ms:.3f} ms |",
           f"| dram__bytes_read.sum + dram__bytes_write.sum | {rd / 1e9:.3f} GB + {wr / 1e9:.3f} GB = {(rd + wr) / 1e9:.3f} GB |",
           f"| DRAM throughput | {(rd + wr) / t_ms / 1e6:.1f} GB/s |"]
    if bt:
        out.append(f"| algorithmic bytes (B_touched) | {bt / 1e9:.3f} GB -> traffic / algorithmic = {(rd + wr) / bt:.2f} |")
    for k, lab in (("lts__t_sector_hit_rate.pct", "L2 sector hit rate"), ("l1tex__t_sector_hit_rate.pct", "L1 sector hit rate"),
                   ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput (% of peak)"),
                   ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active (%)"),
                   ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active (% of peak)"),
                   ("launch__registers_per_thread", "registers / thread"),
                   ("sass__inst_executed_register_spilling", "spill instructions executed"),
                   ("smsp__inst_executed.sum", "warp instructions executed")):
        if k in d:
            out.append(f"| {lab} (`{k}`) | {d[k][0]} {d[k][1]} |")
    out.append(f"| L2 atomic sectors (`lts__t_sectors_srcunit_tex_op_atom.sum`) | {atom:,.0f} -> {atom / t_ms / 1e6:.2f} sectors/ns |")
    for k in ("lts__t_sectors_srcunit_tex_op_atom.avg.pct_of_peak_sustained_elapsed",
              "lts__average_t_sector_srcunit_tex_op_atom_hit_rate.pct"):
        if k in d:
            out.append(f"| `{k}` | {d[k][0]} {d[k][1]} |")
    st = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
    tot = sum(float(d[h][0].replace(",", "") or 0) for h in st)
    top = sorted(((float(d[h][0].replace(",", "") or 0), h) for h in st), reverse=True)[:8]
    out += ["", "Warp-stall samples (pc sampling, all samples):", "",
            "| reason | share |", "|---|---|"]
    out += [f"| {h.replace('smsp__pcsamp_warps_issue_stalled_', '')} | {100 * v / tot:.1f} % |" for v, h in top]
    print("\n".join(out))


if __name__ == "__main__":
    main()
