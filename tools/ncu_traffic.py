"""Write profiles/roofline_traffic.json (bench.py's roofline.traffic) from an `ncu --set full`
capture of the layer-1 and layer-2 k_dqgemv launches of the default workload:
    python tools/ncu_traffic.py gpurun_out/gemv_full.ncu-rep profiles/roofline_traffic.json"""
import csv
import io
import json
import subprocess
import sys


def main(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    units = rows[1]
    launches = []
    for r in rows[2:]:
        if "k_dqgemv" not in r[h.index("Kernel Name")]:
            continue
        rd = float(r[h.index("dram__bytes_read.sum")])
        wr = float(r[h.index("dram__bytes_write.sum")])
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd *= scale[units[h.index("dram__bytes_read.sum")]]
        wr *= scale[units[h.index("dram__bytes_write.sum")]]
        launches.append({"dram_read_bytes": rd, "dram_write_bytes": wr,
                         "duration_us": float(r[h.index("gpu__time_duration.sum")])})
    d = {"source": rep.split("/")[-1], "what": "dram__bytes_read.sum + dram__bytes_write.sum per k_dqgemv launch "
         "(layer 1, layer 2) of Llama-70B TP=1 M=16, ncu --set full --clock-control none",
         "launches": launches,
         "traffic_bytes_per_launch": sum(l["dram_read_bytes"] + l["dram_write_bytes"] for l in launches) / len(launches)}
    with open(out, "w") as f:
        json.dump(d, f, indent=1)
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
