"""Summarise an ncu launch list of `python bench.py --steps K --warmup W` into
profiles/traffic.json's kv_step_kernel.decode_population (the bench's roofline.traffic):
the timed region is the LAST K kv_step_kernel launches of the list.
  python tools/traffic_from_launches.py <launches.csv> <K> <name-of-the-committed-csv>"""
import csv
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    path, K, committed = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    rows = defaultdict(dict)
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if "kv_step_kernel" not in r["Kernel Name"]:
            continue
        v = float(r["Metric Value"].replace(",", ""))
        rows[int(r["ID"])][r["Metric Name"]] = v
    ids = sorted(rows)[-K:]
    la = [{"launch": i, "duration_ns": rows[i]["gpu__time_duration.sum"],
           "dram_read": int(rows[i]["dram__bytes_read.sum"]),
           "dram_write": int(rows[i]["dram__bytes_write.sum"])} for i in ids]
    rd = sum(x["dram_read"] for x in la) / K
    wr = sum(x["dram_write"] for x in la) / K
    tj = os.path.join(ROOT, "profiles", "traffic.json")
    d = json.load(open(tj))
    ks = d["kv_step_kernel"]
    old = ks.get("decode_population")
    if old:
        tag = os.path.basename(old.get("capture", "prev")).replace(".csv", "").split("_")[-1]
        ks["decode_population_" + tag] = old
    ks["decode_population"] = {
        "what": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                "--clock-control none over EVERY kv_step_kernel launch of `python bench.py "
                f"--steps {K} --warmup 5` ({committed}); the timed region is the last {K} "
                "launches. ncu serialises launches and flushes caches between them: compare "
                "shares, not absolutes",
        "capture": committed,
        "n_launches": K,
        "traffic": int(rd + wr), "dram_read": int(rd), "dram_write": int(wr),
        "ncu_duration_us_avg": round(sum(x["duration_ns"] for x in la) / K / 1e3, 2),
        "launches": la,
        "note": old.get("note") if old else None}
    json.dump(d, open(tj, "w"), indent=1)
    print(json.dumps({k: v for k, v in ks["decode_population"].items() if k != "launches"}))


if __name__ == "__main__":
    main()
