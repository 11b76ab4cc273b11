"""Rewrites DESIGN.md §6's measurement table and the reference-arm sentence from the bench lines
under profiles/r02_bench/ (the kernel column is kept as written). Runs here."""
import json
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def L(f):
    return json.loads(open(os.path.join(ROOT, "profiles", "r02_bench", f)).read().strip().splitlines()[-1])


p = os.path.join(ROOT, "DESIGN.md")
s = open(p).read()
i = s.index("| config, timed window | node-updates/s |")
j = s.index("The reference arm (`bench.py --impl reference`, config 5, 16 host threads)")
old_rows = s[i:j].strip().splitlines()
kern = {}
for r in old_rows[2:]:
    cells = [c.strip() for c in r.strip().strip("|").split("|")]
    kern[cells[0]] = cells[-1]
rows = [("**5: 4096 × 128², the driver's form `--steps 20 --warmup 5`**", "cfg5_s20.json", True),
        ("5: default `bench.py` (300 steps, the config's own length)", "cfg5.json", False),
        ("4: 8192², 20 steps", "cfg4_s20.json", False), ("4: 8192², 200 steps", "cfg4.json", False),
        ("2: 64 × 256², 1000 steps", "cfg2.json", False),
        ("3: 1024² + sphere, 500 steps", "cfg3.json", False), ("1: 32², 100 steps", "cfg1.json", False)]
out = old_rows[0] + "\n" + old_rows[1] + "\n"
for name, f, bold in rows:
    d = L(f)
    v, e, c, ms = d["value"], d["e2e"]["value"], d["cpu_baseline"]["value"], d["ms_per_step"]
    t = ("%.3f ms/step" % ms) if ms > 0.1 else ("%.1f µs/step" % (ms * 1e3))
    frac = "%.1f%%" % (100 * d["roofline"]["frac"]) if d["roofline"]["frac"] > 0.01 else "—"
    b = "**" if bold else ""
    rat = ("%.0f× / %.0f×" % (v / c, e / c)) if v / c > 20 else ("%.1f× / %.1f×" % (v / c, e / c))
    k = re.sub(r" \((sw_power_cap|SM clock).*?\)$", "", kern[name])
    clk = d["clocks"]
    note = ""
    if clk.get("reasons"):
        note = " (%s, SM clock down to %d MHz)" % (", ".join(clk["reasons"]), clk["sm_min_mhz"])
    elif clk.get("sm_min_mhz", 1965) < 1900:
        note = " (SM clock down to %d MHz)" % clk["sm_min_mhz"]
    out += "| %s | %s%.3e%s (%s) | %s%s%s | %.3e | %.2e → %s%s%s | %s%s |\n" % (
        name, b, v, b, t, b, frac, b, e, c, b, rat, b, k, note)
s = s[:i] + out + "\n" + s[j:]
r1, r2 = L("reference_cfg5.json")["value"], L("reference_cfg5_s20.json")["value"]
s = re.sub(r"The reference arm \(`bench.py --impl reference`, config 5, 16 host threads\): [0-9.e+]+ "
           r"node-updates/s\nin the default form, [0-9.e+]+ in the driver's form",
           "The reference arm (`bench.py --impl reference`, config 5, 16 host threads): %.2e "
           "node-updates/s\nin the default form, %.2e in the driver's form" % (r1, r2), s)
open(p, "w").write(s)
print(out)
