"""Summarise ncu outputs into profiles/ (committed evidence).

usage:
  python tools/ncu_summary.py launches <launches.csv> <out.txt>
  python tools/ncu_summary.py full <report.ncu-rep> <out.txt> [traffic_key]
  python tools/ncu_summary.py dram <metrics.csv> <out.txt>   (tools/ncu_mapbuild.sh: per-launch DRAM bytes)
The `full` mode also records dram bytes per launch of the captured kernel into
profiles/traffic.json under traffic_key (e.g. outdoor/culled/stride1), which bench.py reports
as roofline.traffic.
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3}

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "smsp__sass_inst_executed_op_global_ld.sum",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "lts__t_sectors_srcunit_tex_op_read.sum",
    "smsp__pcsamp_warps_issue_stalled_long_scoreboard", "smsp__pcsamp_warps_issue_stalled_wait",
    "smsp__pcsamp_warps_issue_stalled_short_scoreboard", "smsp__pcsamp_warps_issue_stalled_not_selected",
    "smsp__pcsamp_warps_issue_stalled_selected", "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle",
    # SURVEY §8(d) metric 3: FP32-pipe thread instructions per cycle over the chip's FP32 peak
    "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum.per_cycle_elapsed",
    "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum.per_cycle_elapsed",
    "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum.per_cycle_elapsed",
    "sm__sass_thread_inst_executed_op_ffma_pred_on.sum.peak_sustained",
]


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in data:
        if len(r) <= iv:
            continue
        name = r[ik].split("(")[0].replace("void ", "")
        ms = float(r[iv].replace(",", "")) * SCALE.get(r[iu], 1e-6)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ms
    tot = sum(a[1] for a in agg.values())
    lines = [f"# ncu launch list ({os.path.basename(path)}): gpu__time_duration per kernel, cold-cache, serialised",
             f"# {sum(a[0] for a in agg.values())} launches, {tot:.3f} ms total", ""]
    for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{k[:72]:72s} launches={n:3d} ms={ms:9.4f} share={ms / tot * 100:5.1f}%")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:12]))


def full(rep, out, key=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    hdr, units = r[0], r[1]
    lines = [f"# ncu --set full summary of {os.path.basename(rep)}"]
    traffic = {}
    for vals in r[2:]:
        name = vals[hdr.index("Kernel Name")].split("(")[0]
        lines.append(f"\n## {name}")
        got = {}
        for w in METRICS:
            if w in hdr:
                i = hdr.index(w)
                lines.append(f"{w:60s} {units[i]:10s} {vals[i]}")
                got[w] = (units[i], vals[i])
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        b = 0.0
        for w in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            if w in got:
                u, v = got[w]
                b += float(v.replace(",", "")) * mult.get(u, 1)
        short = name.split("::")[-1].split("<")[0]
        num = lambda w: float(got[w][1].replace(",", "")) if w in got else None
        traffic[short] = {"dram_bytes": b, "warp_inst": num("smsp__inst_executed.sum"),
                          "fma_pipe_pct": num("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
                          "issue_active_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                          "ms": num("gpu__time_duration.sum"),
                          # L2 -> SM read bytes (32-byte sectors requested by the SMs' texture/LSU path)
                          "l2_read_bytes": (32.0 * num("lts__t_sectors_srcunit_tex_op_read.sum")
                                            if num("lts__t_sectors_srcunit_tex_op_read.sum") else None)}
        fp = [w for w in METRICS if "thread_inst_executed_op_f" in w and "per_cycle_elapsed" in w]
        pk = "sm__sass_thread_inst_executed_op_ffma_pred_on.sum.peak_sustained"
        if all(w in got for w in fp) and pk in got:
            ops = sum(float(got[w][1].replace(",", "")) for w in fp)
            peak = float(got[pk][1].replace(",", ""))
            lines.append(f"{'scalar FP32 thread instr / FP32 peak (packed f32x2 not counted)':60s} {'%':10s} "
                         f"{100.0 * ops / peak:.2f}")
    # hottest CUDA source lines (instructions executed, warp stall samples): needs -lineinfo
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur, rows = None, []
    for r in csv.reader(io.StringIO(src)):
        if r and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if not r or not r[0].isdigit():
            continue
        try:
            rows.append((float(r[7] or 0), float(r[4] or 0), cur, int(r[0]), r[1].strip()[:80]))
        except (ValueError, IndexError):
            pass
    if rows:
        ti = sum(x[0] for x in rows) or 1.0
        ts = sum(x[1] for x in rows) or 1.0
        lines.append("\n## hottest source lines: share of instructions executed, share of stall samples")
        for n, st, f, ln, txt in sorted(rows, reverse=True)[:25]:
            lines.append(f"{n / ti * 100:5.1f}% inst {st / ts * 100:5.1f}% stall  {f}:{ln}  {txt}")
    # the L1 load path by source line: global tag requests and shared-memory wavefronts (both take
    # l1tex LSU data-pipe wavefronts, the kernel's co-limit)
    cur, hdr, lsu = None, None, []
    for r in csv.reader(io.StringIO(src)):
        if r and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if not r or not r[0].isdigit() or hdr is None:
            continue
        try:
            tag = float(r[hdr.index("L1 Tag Requests Global")] or 0)
            shw = float(r[hdr.index("L1 Wavefronts Shared")] or 0)
            l2s = float(r[hdr.index("L2 Theoretical Sectors Global")] or 0)
        except (ValueError, IndexError):
            continue
        if tag or shw:
            lsu.append((tag + shw, tag, shw, l2s, cur, int(r[0]), r[1].strip()[:72]))
    if lsu:
        tt = sum(x[1] for x in lsu) or 1.0
        tw = sum(x[2] for x in lsu) or 1.0
        lines.append(f"\n## L1 load path by source line: global tag requests {tt:.3g} (share), shared wavefronts "
                     f"{tw:.3g} (share), L2 sectors")
        for tot, tag, shw, l2s, f, ln, txt in sorted(lsu, reverse=True)[:20]:
            lines.append(f"{tag / tt * 100:5.1f}% tag {shw / tw * 100:5.1f}% shw {l2s:9.3g} sec  {f}:{ln}  {txt}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if key:
        tpath = os.path.join(ROOT, "profiles", "traffic.json")
        t = json.load(open(tpath)) if os.path.exists(tpath) else {}
        t.setdefault(key, {}).update(traffic)
        json.dump(t, open(tpath, "w"), indent=1, sort_keys=True)


def dram(path, out):
    """Per-launch duration and DRAM bytes of a `--metrics` capture (cold-cache, serialised launches)."""
    rows = list(csv.reader(open(path)))
    h0 = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[h0]
    ix = {k: i for i, k in enumerate(hdr)}
    per = collections.OrderedDict()
    for r in rows[h0 + 1:]:
        if len(r) < len(hdr):
            continue
        per.setdefault((int(r[ix["ID"]]), r[ix["Kernel Name"]].split("(")[0]), {})[r[ix["Metric Name"]]] = (
            r[ix["Metric Unit"]], float(r[ix["Metric Value"]].replace(",", "")))
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6,
            "us": 1e-6, "msecond": 1e-3, "ms": 1e-3}
    lines = [f"# per-launch DRAM traffic ({os.path.basename(path)}; ncu --metrics, cold cache, serialised)",
             f"{'id':>4s} {'kernel':44s} {'us':>8s} {'rd MB':>8s} {'wr MB':>8s} {'TB/s':>6s}"]
    for (i, name), m in per.items():
        g = lambda k: m[k][1] * mult.get(m[k][0], 1) if k in m else 0.0
        t, rd, wr = g("gpu__time_duration.sum"), g("dram__bytes_read.sum"), g("dram__bytes_write.sum")
        lines.append(f"{i:4d} {name.split('::')[-1][:44]:44s} {t * 1e6:8.1f} {rd / 1e6:8.1f} {wr / 1e6:8.1f} "
                     f"{(rd + wr) / t / 1e12 if t else 0:6.2f}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:30]))


if __name__ == "__main__":
    if sys.argv[1] == "dram":
        dram(sys.argv[2], sys.argv[3])
    elif sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
