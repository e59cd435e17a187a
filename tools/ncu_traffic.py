"""Per-launch DRAM traffic of the two dominant kernels from an `ncu --set full` capture
of one cfg2 approximation -> profiles/<tag>_ncu_traffic.json (read by bench.py for the
roofline's `traffic` field).  Usage: python tools/ncu_traffic.py rep.ncu-rep out.json"""
import csv
import io
import json
import subprocess
import sys

SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
TSCALE = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
ix = {k: hdr.index(k) for k in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum")}
best = {}
for r in rows[2:]:
    name = r[ix["Kernel Name"]]
    ms = float(r[ix["gpu__time_duration.sum"]]) * TSCALE[units[ix["gpu__time_duration.sum"]]]
    rd = float(r[ix["dram__bytes_read.sum"]]) * SCALE[units[ix["dram__bytes_read.sum"]]]
    wr = float(r[ix["dram__bytes_write.sum"]]) * SCALE[units[ix["dram__bytes_write.sum"]]]
    base = name.split("(")[0]
    if "k_oe_err" in base or ("qgemm_kernel" in base and base.rstrip(")").endswith("1>")):
        key = "error"      # INT8 digit-slice error kernel, or the FP64 EPI_ERR GEMM (qgemm_kernel<.., 1>)
    elif "k_oz_gemm" in base or "qgemm_kernel" in base:
        key = "gemm"       # INT8 modular GEMM of Y = X Q_R, or the FP64 one
    else:
        continue
    if key not in best or ms > best[key]["ms"]:
        best[key] = {"kernel": name.split("(")[0].replace("void ", ""), "ms": ms, "dram_read_bytes": rd,
                     "dram_write_bytes": wr, "traffic_bytes": rd + wr}
json.dump({"source": rep, "note": "largest launch of each kind in one cfg2 approximation, ncu --set full",
           "gemm_xq": best.get("gemm"), "error": best.get("error")}, open(out, "w"), indent=1)
print(json.dumps(best, indent=1))
