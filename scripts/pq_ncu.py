#!/usr/bin/env python
"""Device time per LaB-PQ call from an ncu launch list of scripts/pq_bench.py.

  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file L.csv python scripts/pq_bench.py
  python scripts/pq_ncu.py L.csv
Prints every sssp::pq_* launch in order with its duration (the pq_bench call order tells
which call each belongs to) and the per-kernel-name totals of the last occurrence groups.
"""
import csv
import sys

rows = [r for r in csv.DictReader(ln for ln in open(sys.argv[1]) if ln.startswith('"'))
        if r.get("Metric Name") == "gpu__time_duration.sum" and "pq_" in r.get("Kernel Name", "")]
for r in rows:
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "")
    us = v / 1e3 if unit in ("nsecond", "ns") else (v if unit in ("usecond", "us") else v * 1e3)
    print(f"{r['ID']:>5} {r['Kernel Name'].split('(')[0]:40s} {us:9.2f} us")
