"""profiles/traffic.json from an ncu --set full capture of the fused forward (tools/gpu_final.sh):
per weighted layer, dram__bytes_read.sum + dram__bytes_write.sum of its launch, plus the
tensor-pipe and DRAM utilisation ncu reports. Launch i of the capture is weighted layer i."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LAYERS = [0, 4, 9, 13, 18, 22, 27, 31, 35]  # weighted layers of the default network, launch order


def main(rep, batch):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    out = {}
    kn = hdr.index("Kernel Name")
    layer_rows = [r for r in rows[2:] if "prep_" not in r[kn]]  # build-time weight preparation: not a layer
    for i, r in enumerate(layer_rows[:len(LAYERS)]):
        d = dict(zip(hdr, r))

        def num(k):
            try:
                return float(d[k].replace(",", ""))
            except (KeyError, ValueError):
                return None
        unit = rows[1][hdr.index("dram__bytes_read.sum")]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
        out[f"layer{LAYERS[i]}"] = {
            "kernel": d.get("Kernel Name", "")[:80],
            "traffic_bytes": (rd + wr) * scale if rd is not None and wr is not None else None,
            "duration_us": num("gpu__time_duration.sum"),
            "tensor_pipe_pct": num("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
            "dram_pct": num("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "sm_throughput_pct": num("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
        }
    path = os.path.join(ROOT, "profiles", "traffic.json")
    allb = json.load(open(path)) if os.path.exists(path) else {}
    allb[f"b{batch}"] = {k: v["traffic_bytes"] for k, v in out.items()}
    allb[f"b{batch}_detail"] = out
    json.dump(allb, open(path, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 256)
