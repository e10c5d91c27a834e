"""Copy a profile_round.sh bundle from gpurun_out/ into profiles/ (ROUND, default r2):
bench line, launch list, ncu summaries, traffic.json and the SASS of the
dominant kernels.  Run here after the GPU call.

    python tools/update_profiles.py
"""
import json
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
sys.path.insert(0, ROOT)


def summary(rep, first=None):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep],
                         capture_output=True, text=True).stdout
    blocks = ["==" + b for b in out.split("==")[1:] if b.strip()]
    return "".join(blocks[:first] if first else blocks)


def raw_bytes(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout.splitlines()
    import csv
    rows = list(csv.reader(out))
    h = {k: i for i, k in enumerate(rows[0])}
    res = []
    for r in rows[2:]:
        rd, wr = float(r[h["dram__bytes_read.sum"]]), float(r[h["dram__bytes_write.sum"]])
        unit_r, unit_w = rows[1][h["dram__bytes_read.sum"]], rows[1][h["dram__bytes_write.sum"]]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        res.append((r[h["Kernel Name"]], int(rd * scale[unit_r] + wr * scale[unit_w])))
    return res


R = os.environ.get("ROUND", "r2")
shutil.copy(os.path.join(G, "bench.json"), os.path.join(P, f"{R}_bench.json"))
shutil.copy(os.path.join(G, "launches.csv"), os.path.join(P, f"{R}_bench_launches.csv"))
with open(os.path.join(P, f"{R}_ncu_summary.txt"), "w") as fh:
    fh.write(f"# {R}: ncu --set full --clock-control none, one launch per kernel "
             "(cold-cache replays: the kernel's share of the step, not its absolute time)\n")
    fh.write("# C2 frame kernel (k_pair3<1,0>, 640K nodes)\n" + summary(os.path.join(G, "c2_frame.ncu-rep"), 1))
    fh.write("# C5 fused frame kernel (k_pair3<1,0>, 16.8M nodes)\n" + summary(os.path.join(G, "c5_frame.ncu-rep"), 1))
    fh.write("# C5 split passes: stand-alone k_pair_normals, then force+integrate k_pair3<0,0>\n" + summary(os.path.join(G, "c5_split.ncu-rep"), 2))
    fh.write("# C3 collision (draped: after 200 frames): fused narrow phase + respond\n" + summary(os.path.join(G, "c3_draped.ncu-rep")))
    if os.path.exists(os.path.join(G, "c2_fixed.ncu-rep")):
        fh.write("# C2 reference-exact (fixed) pair: k_pair_normals_x, then the guarded exact force pass k_pair3<0,0,0,1>\n" + summary(os.path.join(G, "c2_fixed.ncu-rep"), 2))
    if os.path.exists(os.path.join(G, "band8.ncu-rep")):
        fh.write("# 8-way band of C5 (516 local rows), self-linked: BAND k_pair3 with peer stores + in-kernel seam handshake\n" + summary(os.path.join(G, "band8.ncu-rep"), 1))
t = {"_source": f"ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum per launch "
                f"(profiles/{R}_ncu_summary.txt): C2 / C5_frame = fused k_pair3<1,0>, "
                "C5 = k_pair3<0,0> force pass, C5_normals = k_pair_normals, C3_detect = the "
                "fused narrow phase of a draped C3 frame"}
t["C2"] = raw_bytes(os.path.join(G, "c2_frame.ncu-rep"))[0][1]
t["C5_frame"] = raw_bytes(os.path.join(G, "c5_frame.ncu-rep"))[0][1]
for name, b in raw_bytes(os.path.join(G, "c5_split.ncu-rep")):
    if "normals" in name:
        t.setdefault("C5_normals", b)
    else:
        t.setdefault("C5", b)
for name, b in raw_bytes(os.path.join(G, "c3_draped.ncu-rep")):
    if "detect" in name:
        t.setdefault("C3_detect", b)
json.dump(t, open(os.path.join(P, "traffic.json"), "w"), indent=2)
print(json.dumps(t, indent=1))

lib = os.path.join(ROOT, "paper_2507_11794_b200", "_lib", "libclothsim_b200.so")
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
want = {"k_pair3ILb1ELb0ELb0ELb0ELb0E": f"{R}_sass_k_pair3_fused.txt",
        "k_pair3ILb0ELb0ELb0ELb0ELb0E": f"{R}_sass_k_pair3_force.txt",
        "k_pair3ILb0ELb0ELb0ELb1ELb0E": f"{R}_sass_k_pair3_exact.txt",
        "k_pair3ILb1ELb0ELb0ELb0ELb1E": f"{R}_sass_k_pair3_band.txt",
        "k_detect_tri": f"{R}_sass_k_detect_tri.txt"}
for part in sass.split("Function : ")[1:]:
    name = part.split("\n", 1)[0]
    for k, f in want.items():
        if k in name:
            out = []
            for line in part.split("\n"):
                if re.match(r"^\s+/\* 0x[0-9a-f]+ \*/$", line) or not line.strip():
                    continue
                line = re.sub(r"\s+/\* 0x[0-9a-f]+ \*/$", "", line.rstrip())
                out.append(re.sub(r"\s{2,}", " ", line))
            open(os.path.join(P, f), "w").write("Function : " + "\n".join(out) + "\n")
