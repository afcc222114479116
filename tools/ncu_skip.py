"""Prints `-s S -c C` for ncu so a --set full capture covers exactly the LAST pass of a
tools/prof_workload.py run (warm-up pass + 1 rep): counts the launches matching the regex
in the launch list of the same command and skips the first half."""
import csv
import re
import sys

rows = []
with open(sys.argv[1]) as f:
    lines = [ln for ln in f if ln.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") == "gpu__time_duration.sum" and re.search(sys.argv[2], r["Kernel Name"]):
        rows.append(r["ID"])
n = len(set(rows))
print(f"-s {n // 2} -c {n - n // 2}")
