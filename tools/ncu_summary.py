"""Compact summary of ncu --set full reports (.ncu-rep) for profiles/.

    python tools/ncu_summary.py out.json a.ncu-rep [b.ncu-rep ...]
    python tools/ncu_summary.py --traffic profiles/traffic.json "key=rep.ncu-rep" ...
(the second form records per-launch DRAM bytes under the keys bench.py looks up)

Per report and kernel: duration, DRAM bytes read/written (the `traffic` of
bench.py's roofline), throughputs, tensor-pipe activity, L2 hit rate,
occupancy, registers.
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "lts__t_bytes.sum": "l2_bytes",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__registers_per_thread": "regs",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:90]}
        for i, (h, u) in enumerate(zip(hdr, units)):
            key = next((v for k, v in KEYS.items() if h == k or h.endswith("." + k)), None)
            if key is None or key in d:
                continue
            try:
                val = float(r[i].replace(",", ""))
            except ValueError:
                continue
            d[key] = val * SCALE.get(u, 1)
        if "duration" in d:
            d["duration_us"] = d.pop("duration")
        if "dram_read" in d and "dram_write" in d:
            d["dram_bytes"] = d["dram_read"] + d["dram_write"]
            d["dram_GBps"] = d["dram_bytes"] / (d["duration_us"] * 1e-6) / 1e9
        res.append(d)
    return res


if __name__ == "__main__":
    if sys.argv[1] == "--traffic":
        out = {}
        for kv in sys.argv[3:]:
            key, rep = kv.rsplit("=", 1)
            d = summarise(rep)[0]
            out[key] = {"dram_bytes": d.get("dram_bytes"), "duration_us": d.get("duration_us"),
                        "source": rep.rsplit("/", 1)[-1]}
        json.dump(out, open(sys.argv[2], "w"), indent=1)
        print(json.dumps(out, indent=1))
        sys.exit(0)
    allr = {}
    for rep in sys.argv[2:]:
        allr[rep.rsplit("/", 1)[-1]] = summarise(rep)
    json.dump(allr, open(sys.argv[1], "w"), indent=1)
    for k, v in allr.items():
        for d in v:
            print(k, json.dumps({a: (round(b, 2) if isinstance(b, float) else b) for a, b in d.items()}))
