#!/usr/bin/env python
"""Summarise an ncu --csv launch list of tools/nvlink_group_ncu.py: per
step kernel and device, NVLink tx/rx bytes (all and user data, 32-byte
granularity) against the algorithmic push bytes the tool printed.

  python tools/nvlink_summary.py gpurun_out/r02z_nvlink_g2.csv gpurun_out/r02z_plain_g2.log"""
from __future__ import annotations

import collections
import csv
import json
import re
import sys

METRICS = ["gpu__time_duration.sum", "nvltx__bytes.sum", "nvltx__bytes_data_user.sum",
           "nvlrx__bytes.sum", "nvlrx__bytes_data_user.sum", "dram__bytes_read.sum", "dram__bytes_write.sum"]


def main() -> None:
    rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
    h = rows[0]
    ix = {k: h.index(k) for k in h}
    plain = {}
    if len(sys.argv) > 2:
        for line in open(sys.argv[2]):
            if line.startswith("{"):
                plain = json.loads(line)
    launches = collections.OrderedDict()
    for r in rows[1:]:
        name = re.sub(r"\(.*", "", r[ix["Kernel Name"]]).replace("void ", "").replace("unnamed>::", "")
        if not re.search(r"k1_gather|k_shard_p2p", name):
            continue
        key = (int(r[ix["ID"]]), int(r[ix["Device"]]), name)
        launches.setdefault(key, {})[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
    G = plain.get("G") or len({d for _, d, _ in launches})
    steps = sum(1 for (_, d, k) in launches if d == 0 and k.startswith("k1_gather"))
    per = collections.defaultdict(lambda: collections.defaultdict(float))  # (kernel, device) -> sums per step
    for (_, d, k), v in launches.items():
        fam = "K1 push (k1_gather)" if k.startswith("k1_gather") else "shard update (k_shard_p2p, all buckets)"
        for m in METRICS:
            per[(fam, d)][m] += v.get(m, 0.0) / steps
        per[(fam, d)]["launches"] += 1 / steps
    alg = plain.get("algorithmic_per_rank", {})
    out = {"G": G, "workload": plain.get("workload"), "n": plain.get("n"), "steps_profiled": steps,
           "algorithmic_tx_bytes_per_rank": {"K1 push (k1_gather)": alg.get("K1_push_tx_bytes"),
                                             "shard update (k_shard_p2p, all buckets)": alg.get("shard_weight_push_tx_bytes")},
           "per_rank_per_step": []}
    for (fam, d), v in sorted(per.items()):
        a = out["algorithmic_tx_bytes_per_rank"][fam]
        t = v["gpu__time_duration.sum"] * 1e-9
        out["per_rank_per_step"].append({
            "kernel": fam, "device": d, "launches": round(v["launches"], 2),
            "time_us": round(t * 1e6, 1),
            "nvl_tx_bytes": v["nvltx__bytes.sum"], "nvl_tx_user_bytes": v["nvltx__bytes_data_user.sum"],
            "nvl_rx_bytes": v["nvlrx__bytes.sum"], "nvl_rx_user_bytes": v["nvlrx__bytes_data_user.sum"],
            "tx_user_over_algorithmic": round(v["nvltx__bytes_data_user.sum"] / a, 4) if a else None,
            "tx_wire_GBps": round(v["nvltx__bytes.sum"] / t / 1e9, 1) if t else None,
            "dram_bytes": v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"],
            "dram_GBps": round((v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"]) / t / 1e9, 1) if t else None})
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
