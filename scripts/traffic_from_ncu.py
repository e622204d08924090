"""Build profiles/<round>_traffic.json from an ncu --set full capture of one bsf_eval_all_batch call
(k_frame, k_band, k_core): DRAM bytes per algorithmic byte (read here with `ncu -i`, no GPU needed).

usage: python scripts/traffic_from_ncu.py gpurun_out/core_full.ncu-rep 20 profiles/r01_traffic.json [core_cps]
core_cps: control points of the core rectangle (C2: 120 x 120 = 14400) for k_core's own ratio.
"""
import csv, io, json, subprocess, sys, os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

rep, nst, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, data = rows[0], rows[2:]
ik, ir, iw, it = (hdr.index(k) for k in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum",
                                          "gpu__time_duration.sum"))
units = rows[1]
scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
kern = {}
for r in data:
    name = r[ik].split("(")[0].split("::")[-1]
    kern[name] = {"dram_read_MB": float(r[ir]) * scale[units[ir]], "dram_write_MB": float(r[iw]) * scale[units[iw]],
                  "duration_us": float(r[it]) * (1e-3 if units[it] == "nsecond" else 1.0)}
# algorithmic bytes of one call over nst C2 states: positions + gradient 24 B each per
# control point, 72 B per block
import workloads as W
import paper_2506_18867_b200 as B
sh = W.make_c2()
h = B.Sheet.from_sheet(sh, device=-1)
n_cp = sh.n_u * sh.n_v
alg_MB = nst * (48.0 * n_cp + 72.0 * h.nnzb) / 1e6
tot = sum(v["dram_read_MB"] + v["dram_write_MB"] for v in kern.values())
core_cps = int(sys.argv[4]) if len(sys.argv) > 4 else 14400
for name, v in kern.items():
    if name.startswith("k_core"):   # k_core's algorithmic bytes: 48 B per core control point + 23 blocks x 72 B
        v["algorithmic_MB"] = nst * core_cps * (48 + 23 * 72) / 1e6
        v["dram_bytes_per_algorithmic_byte"] = (v["dram_read_MB"] + v["dram_write_MB"]) / v["algorithmic_MB"]
json.dump({"dram_bytes_per_algorithmic_byte": tot / alg_MB,
           "source": f"{rep} (ncu --set full, {', '.join(sorted(kern))} of one call, {nst} C2 states)",
           "kernels": kern, "algorithmic_MB": alg_MB,
           "note": "DRAM bytes below the algorithmic bytes: the last ~tens of MB of each capture are still "
                   "resident in the 126 MB L2 when the kernel ends"}, open(out, "w"), indent=1)
print(open(out).read())
