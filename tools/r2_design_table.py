"""Rewrite DESIGN.md section 9's round-2 summary table and per-config table from
profiles/TAG_bench_default.json and TAG_bench_chained.json.  usage: python tools/r2_design_table.py TAG"""
import json
import re
import sys

tag = sys.argv[1]
b = json.load(open(f"profiles/{tag}_bench_default.json"))
c = json.load(open(f"profiles/{tag}_bench_chained.json"))
po, cb, pc = b["per_op"], b["cpu_baseline"], b["per_config"]
p = "DESIGN.md"
s = open(p).read()
i = s.index("**Round 2 (driver-comparable bench line, `profiles/")
j = s.index("What moved between r2b and")


def step(kern):
    # the transcoders as timed inside the bench step (the launches the roofline line uses)
    k = b["roofline"]["kernels"][kern]
    return f"{k['avg_launch_ms']:.2f} ms ({k['frac']:.3f}, in the step)"


def f(op):
    return f"{po[op]['ms']:.2f} ms ({po[op]['frac_of_peak']:.3f})"


new = f"""**Round 2 (driver-comparable bench line, `profiles/{tag}_bench_default.json`, 8 GiB config 4,
one B200, clocks 1965 MHz, no throttle reasons; interim builds `profiles/r2a_*`, `r2b_*`; r2d–r2g in git history):**

| Step / kernel | round 1 (r1m) | round 2 interim (r2b) | round 2 final two-pass ({tag}) | round 2 single-pass (`--path chained`, {tag}) |
|---|---|---|---|---|
| bench value (input GB/s of both transcoding passes) | 827.5 | 855.2 | **{b['value']:.1f}** | {c['value']:.1f} |
| ms per step | 24.01 | 23.23 | {b['ms_per_step']:.2f} | {c['ms_per_step']:.2f} |
| forward transcoder (8 GiB) | 10.07 ms (0.306) | 9.17 ms (0.336) | {step('k_transcode_planned<U8Pol>')} | {f('utf8_to_utf16le')} |
| reverse transcoder (11.3 GB UTF-16) | 10.85 ms (0.284) | 10.62 ms (0.290) | {step('k_transcode_planned<U16Pol>')} | {f('utf16le_to_utf8')} |
| sizing pass, UTF-8 (len16 / + plan) | 1.31 ms | 1.85 ms (plan) | **{po['plan_utf8 (len16 + plan)']['ms']:.2f} ms (plan)** | {po['utf16_length_from_utf8']['ms']:.2f} ms |
| sizing pass, UTF-16 (len8 / + plan) | 1.57 ms | 1.65 ms (plan) | {po['plan_utf16le (len8 + plan)']['ms']:.2f} ms (plan) | {po['utf8_length_from_utf16le']['ms']:.2f} ms |
| utf8_validate / utf16le_validate | 0.49 / 0.72 | 0.47 / 0.71 | {po['utf8_validate']['frac_of_peak']:.2f} / {po['utf16le_validate']['frac_of_peak']:.2f} | — |
| f4 keyed decoder (forward, planned) | — | — | {f('utf8_to_utf16le_keyed (f4)')} | — |
| DRAM traffic of the transcoders | extrapolated from 1 GiB | measured at 8 GiB: 1.00× | measured at 8 GiB: 1.00× algorithmic | — |
| e2e (host buffers, link-bound) | 40.6 GB/s | 42.2 GB/s | {b['e2e']['value']:.1f} GB/s | — |
| oracle, 16 host threads / 1 pinned thread | 1.56 GB/s / — | 1.96 / 0.12 GB/s | {cb['value']:.2f} / {cb['single_thread']['value']:.2f} GB/s | — |

"""
s = s[:i] + new + s[j:]
s = re.sub(r"What moved between r2b and r2\w \(each A/B", f"What moved between r2b and {tag} (each A/B", s)
s = re.sub(r"\(r2\w; per-call CUDA events, 50 calls", f"({tag}; per-call CUDA events, 50 calls", s)
k0 = s.index("| cfg | utf8_validate | utf8→16 planned | utf8→16 single |")
k1 = s.index("\n\n", k0)
rows = ["| cfg | utf8_validate | utf8→16 planned | utf8→16 single | utf16le_validate | utf16→8 planned | utf16→8 single | plan utf8 | plan utf16 | len16←8 | len8←16 |",
        "|---|---|---|---|---|---|---|---|---|---|---|"]
for key, label in [("c1", "c1 (1 GiB ASCII)"), ("c2a", "c2a (256 MiB)"), ("c2b", "c2b (256 MiB)"),
                   ("c3", "c3 (512 MiB)")]:
    r = pc[key]

    def cell(op):
        return f"{r[op]['input_gbs']:.0f} ({r[op]['frac_of_peak']:.2f})"
    rows.append(f"| {label} | {cell('utf8_validate')} | {cell('utf8_to_utf16le_planned')} | "
                f"{cell('utf8_to_utf16le')} | {cell('utf16le_validate')} | "
                f"{cell('utf16le_to_utf8_planned')} | {cell('utf16le_to_utf8')} | "
                f"{cell('plan_utf8 (len16 + plan)')} | {cell('plan_utf16le (len8 + plan)')} | "
                f"{cell('utf16_length_from_utf8')} | {cell('utf8_length_from_utf16le')} |")
s = s[:k0] + "\n".join(rows) + s[k1:]
open(p, "w").write(s)
print("DESIGN.md section 9 tables from", tag)
