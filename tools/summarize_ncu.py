"""Summarise ncu outputs into profiles/ (launch-list shares + full-capture metrics)."""
import csv, json, subprocess, sys
from collections import defaultdict

def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    out = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "ns")
        scale = {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6}.get(unit, 1e-6)
        out[name][0] += 1
        out[name][1] += v * scale
    tot = sum(v[1] for v in out.values())
    return {k: {"launches": v[0], "ms": round(v[1], 3), "share": round(v[1] / tot, 4)}
            for k, v in sorted(out.items(), key=lambda kv: -kv[1][1])}, tot

def full(rep, kernel_regex):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr = rows[0]
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__grid_size",
            "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio"]
    res = []
    units = rows[1]
    scale = {"Gbyte": 1.0, "Mbyte": 1e-3, "Kbyte": 1e-6, "byte": 1e-9, "ms": 1.0, "msecond": 1.0, "us": 1e-3,
             "usecond": 1e-3, "ns": 1e-6, "nsecond": 1e-6}
    for r in rows[2:]:
        d = {}
        for w in want:
            if w not in hdr:
                continue
            i = hdr.index(w)
            v = r[i]
            if units[i] in scale:  # normalise to GB / ms
                v = repr(float(v.replace(",", "")) * scale[units[i]])
            d[w] = v
        res.append(d)
    return res

if __name__ == "__main__":
    tag = sys.argv[1]
    summ, tot = launches("gpurun_out/launches.csv")
    json.dump({"command": "python bench.py --steps 1 --warmup 1 --no-extra --no-cpu",
               "note": "ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised launches)",
               "total_ms": round(tot, 3), "kernels": summ}, open(f"profiles/{tag}_launches_summary.json", "w"), indent=1)
    kern = sys.argv[2] if len(sys.argv) > 2 else "lu_gemm3m_tma_kernel"
    f = full("gpurun_out/prof_gemm_r1.ncu-rep", kern)
    json.dump({"command": f"ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:{kern}<.int.128' -s 10 -c 1 python bench.py --steps 1 --warmup 1 --no-extra --no-cpu",
               "units": "GB, ms",
               "kernels": f}, open(f"profiles/{tag}_lu_gemm_ncu_full.json", "w"), indent=1)
    g = f[0]
    traffic = (float(g["dram__bytes_read.sum"]) + float(g["dram__bytes_write.sum"])) * 1e9  # GB -> bytes
    json.dump({kern: {"bytes_per_launch": traffic,
                                      "launch": f"11th rank-128 trailing update ({kern}<128>, super-panel k = 10*128) of cfg2",
                                      "gpu_time_ms": float(g["gpu__time_duration.sum"])}},
              open("profiles/ncu_traffic.json", "w"), indent=1)
    print(json.dumps(summ, indent=0)[:1500])
