"""Print one precond apply (+ J apply) from an ncu launch list of tools/profile_apply.py.

    python tools/apply_segment.py gpurun_out/launch_apply_cfg3.csv [out.txt]
"""
import sys

sys.path.insert(0, "tools")
import launches as L  # noqa: E402

d = L.load(sys.argv[1])
starts = [i for i, k in enumerate(d) if "hsolve_in" in k["name"]]
s = starts[2] if len(starts) > 2 else starts[-1]
e = starts[3] if len(starts) > 3 else s + 34
seg = d[s:e] if e - s < 60 else d[s:s + 34]
tot, out = 0.0, []
for k in seg:
    t = k["gpu__time_duration.sum"] / 1e3
    tot += t
    rd, wr = k["dram__bytes_read.sum"] / 1e6, k["dram__bytes_write.sum"] / 1e6
    out.append(f"{t:8.1f} us rd {rd:8.2f} MB wr {wr:7.2f} MB {(rd + wr) / t if t else 0:5.2f} TB/s  "
               f"{L.short(k)} {k['grid']}")
out.append(f"total {tot:.1f} us over {len(seg)} launches (precond apply + J apply)")
txt = "\n".join(out) + "\n"
print(txt)
if len(sys.argv) > 2:
    open(sys.argv[2], "w").write(txt)
