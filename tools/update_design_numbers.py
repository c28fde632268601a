"""Refresh the measured numbers in DESIGN.md section 9 (per-op table, all-config table, bench
paragraph head, file references) from a measurement round.
usage: python tools/update_design_numbers.py TAG PREV_TAG"""
import json
import re
import sys

tag, prev = sys.argv[1], sys.argv[2]
rows = json.load(open(f"profiles/{tag}_ops_allcfg.json"))
ops = ["utf8_validate", "utf8_to_utf16le", "utf16le_validate", "utf16le_to_utf8",
       "utf16_length_from_utf8", "utf8_length_from_utf16le", "utf8_to_utf16be", "utf16be_to_utf8"]
tbl = "\n".join(f"| {r['cfg']} ({r['mib']}) | " + " | ".join(
    f"{r[o]['in_gbs']:.0f} ({r[o]['frac']:.2f})" for o in ops) + " |" for r in rows) + "\n"
d = json.load(open(f"profiles/{tag}_bench_default.json"))
K = d["roofline"]["kernels"]
f, r = K["k_transcode<U8Pol>"], K["k_transcode16"]
sh = open(f"profiles/{tag}_ncu_launches.txt").read()
shf = float(re.search(r"k_transcode<U8PolT<0>>.*?([\d.]+)\s*$", sh, re.M).group(1))
shr = float(re.search(r"k_transcode16<0>.*?([\d.]+)\s*$", sh, re.M).group(1))
s = open("DESIGN.md").read()
n0 = len(s)


def rep(old, new):
    global s
    assert s.count(old) == 1, old[:70]
    s = s.replace(old, new)


a = s.index("| cfg (MiB) | utf8_validate |")
b = s.index("(c2a / c2b / c3 are 256–512 MiB")
assert 0 < a < b
he = s.index("\n", s.index("|---|", a)) + 1
s = s[:he] + tbl + "\n" + s[b:]
rep(f"`profiles/{prev}_ops_allcfg.json`; input GB/s", f"`profiles/{tag}_ops_allcfg.json`; input GB/s")
c = {x["cfg"]: x for x in rows}
a = s.index("| utf8_to_utf16le (c4) | 474 GB/s (0.17) |")
b = s.index("| utf8_validate (c4) |")
assert 0 < a < b


def cell(cfg, op):
    return f"{c[cfg][op]['in_gbs']:.0f} GB/s ({c[cfg][op]['frac']:.2f})"


s = s[:a] + f"""| utf8_to_utf16le (c4) | 474 GB/s (0.17) | {cell('c4', 'utf8_to_utf16le')} |
| utf16le_to_utf8 (c4) | 418 GB/s (0.11) | {cell('c4', 'utf16le_to_utf8')} |
| utf8_to_utf16le (c1 ASCII) | ≈ 670 GB/s | {cell('c1', 'utf8_to_utf16le')} |
| utf16le_to_utf8 (c1 ASCII) | — | {cell('c1', 'utf16le_to_utf8')} |
| utf16le_to_utf8 (c3 emoji) | — | {cell('c3', 'utf16le_to_utf8')} |
""" + s[b:]
a = s.index(f"Bench step (8 GiB config 4, `profiles/{prev}_bench_default.json`)")
b = s.index("the first r1 line was 664.6), of which", a)
assert 0 < a < b
first, second = (("reverse", r), ("forward", f)) if r["avg_launch_ms"] >= f["avg_launch_ms"] \
    else (("forward", f), ("reverse", r))
s = s[:a] + (f"Bench step (8 GiB config 4, `profiles/{tag}_bench_default.json`): **{d['value']:.1f} "
             f"GB/s** ({d['ms_per_step']:.2f} ms;\n") + s[b:]
a = s.index("the first r1 line was 664.6), of which")
b = s.index("e2e through the host-buffer API", a)
s = s[:a] + (f"the first r1 line was 664.6), of which the {first[0]} transcoder "
             f"{first[1]['avg_launch_ms']:.2f} ms ({first[1]['frac']:.3f} of peak)\nand the "
             f"{second[0]} {second[1]['avg_launch_ms']:.2f} ms ({second[1]['frac']:.3f}) — "
             f"{(shr if first[0] == 'reverse' else shf) * 100:.1f} % / "
             f"{(shf if first[0] == 'reverse' else shr) * 100:.1f} % of the step\n"
             f"(`profiles/{tag}_ncu_launches.txt`); ") + s[b:]
s = re.sub(r"e2e through the host-buffer API [\d.]+ GB/s",
           f"e2e through the host-buffer API {d['e2e']['value']:.1f} GB/s", s, count=1)
s = s.replace(f"Measured on one B200 (`profiles/{prev}_*`,", f"Measured on one B200 (`profiles/{tag}_*`,")
s = s.replace(f"list `profiles/{prev}_ncu_launches.txt` — so the line lists both",
              f"list `profiles/{tag}_ncu_launches.txt` — so the line lists both")
s = s.replace(f"(`profiles/{prev}_ncu_full_transcoders.txt`:", f"(`profiles/{tag}_ncu_full_transcoders.txt`:")
assert 0.9 * n0 < len(s) < 1.1 * n0, (n0, len(s))
open("DESIGN.md", "w").write(s)
t = open("profiles/README.md").read()
t = re.sub(r"\*\*`(r1\w+)` \(current[^)]*\)\*\*", lambda m: f"`{m.group(1)}`", t)
t = t.rstrip().rstrip(".") + f", **`{tag}` (current: {d['value']:.1f} GB/s)**.\n"
open("profiles/README.md", "w").write(t)
print(d["value"], first[0], first[1]["frac"], second[0], second[1]["frac"])
