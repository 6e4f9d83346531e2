"""Attribute ncu warp-stall samples of one kernel to source functions (inlined code included).

usage: python tools/ncu_regions.py report.ncu-rep kernel_regex lib.so [cubin_name_substr] [mangled_fn_regex]
Maps each SASS address of the ncu source page to the innermost file:line that `nvdisasm -g`
reports (build with -lineinfo), then to the enclosing function (the last `__device__` /
`__global__` definition above that line). Prints samples and stall_no_inst per function."""
import collections, csv, glob, os, re, subprocess, sys, tempfile

rep, kern, lib = sys.argv[1], sys.argv[2], sys.argv[3]
cub_sub = sys.argv[4] if len(sys.argv) > 4 else ""
fn_re = sys.argv[5] if len(sys.argv) > 5 else kern  # mangled-name regex of the SASS function, if it differs
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
lines_of = {}
for cub in glob.glob(os.path.join(tmp, "*.cubin")):
    if cub_sub not in os.path.basename(cub):
        continue
    txt = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
    cur, loc = None, None
    for ln in txt.splitlines():
        m = re.match(r"^\.text\.(\S+):", ln)
        if m:
            cur = m.group(1)
            lines_of[cur] = {}
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            loc = (m.group(1), int(m.group(2)))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
        if m and cur:
            lines_of[cur][int(m.group(1), 16)] = loc
fn = [k for k in lines_of if re.search(fn_re, k)]
assert fn, f"no function matching {kern}"
amap = lines_of[fn[0]]
out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kern}", "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
body = [r for r in rows[hi + 1:] if len(r) > 5 and r[0].startswith("0x")]
base = int(body[0][0], 16)
ci = {k: h.index(k) for k in ("Warp Stall Sampling (All Samples)", "stall_no_inst", "stall_wait", "stall_barrier", "L1 Wavefronts Shared", "L1 Wavefronts Shared Excessive",
                              "stall_long_sb", "stall_short_sb", "Instructions Executed")}
func_starts = {}
def func_of(loc):
    if loc is None:
        return "?"
    f, line = loc
    if f not in func_starts:
        starts = []
        try:
            for k, s in enumerate(open(f), 1):
                m = re.match(r"^(?:template.*\n)?\s*(?:static\s+)?(?:__device__|__global__|VHD)[^(]*?\b(\w+)\s*\(", s)
                if m:
                    starts.append((k, m.group(1)))
        except OSError:
            pass
        func_starts[f] = starts
    name = "?"
    for k, n in func_starts[f]:
        if k <= line:
            name = n
    return f"{os.path.basename(f)}:{name}"
agg = collections.defaultdict(lambda: collections.Counter())
for r in body:
    loc = amap.get(int(r[0], 16) - base)
    key = func_of(loc)
    for k, i in ci.items():
        agg[key][k] += float(r[i] or 0)
tot = sum(v["Warp Stall Sampling (All Samples)"] for v in agg.values())
print(f"{fn[0][:80]}\n{len(body)} SASS lines, {tot:.0f} samples")
print(f"{'function':48s} {'samples':>8s} {'share':>6s} {'no_inst':>8s} {'wait':>7s} {'barrier':>8s} {'long_sb':>8s} {'instr':>9s} {'smem_wf':>8s} {'smem_excess':>11s}")
for k, v in sorted(agg.items(), key=lambda x: -x[1]["Warp Stall Sampling (All Samples)"])[:30]:
    s = v["Warp Stall Sampling (All Samples)"]
    print(f"{k[:48]:48s} {s:8.0f} {s / tot:6.1%} {v['stall_no_inst']:8.0f} {v['stall_wait']:7.0f} {v['stall_barrier']:8.0f} "
          f"{v['stall_long_sb']:8.0f} {v['Instructions Executed']:9.0f} {v['L1 Wavefronts Shared']:8.0f} {v['L1 Wavefronts Shared Excessive']:11.0f}")
