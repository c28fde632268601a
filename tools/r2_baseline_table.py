"""Rewrite BASELINE.md section 4 (measured results) from profiles/TAG_bench_default.json.
usage: python tools/r2_baseline_table.py TAG"""
import json
import sys

tag = sys.argv[1]
d = json.loads(open(f"profiles/{tag}_bench_default.json").read())
pc, po, c, cb = d["per_config"], d["per_op"], d["config"], d["cpu_baseline"]
rows = []


def row(cfg, op, in_gbs, gch, hbm, par, o1="—", on="—"):
    rows.append(f"| {cfg} | {op} | 1 | {in_gbs:.0f} | {gch:.0f} | {hbm / 1000:.2f} | "
                f"{100 * hbm / 8000:.0f} % | {100 * hbm / 6452.5:.0f} % | {o1} | {on} | {par} |")


names = {"utf8_to_utf16le_planned": "UTF-8→UTF-16LE (two-pass)",
         "utf16le_to_utf8_planned": "UTF-16LE→UTF-8 (two-pass)",
         "utf8_validate": "utf8_validate", "utf16le_validate": "utf16le_validate"}
par = "bit-exact at full size, both paths (tests/test_gpu_fullsize.py)"
for cfg, label in [("c1", "C1: 1 GiB ASCII"), ("c2a", "C2A: 256 MiB"), ("c2b", "C2B: 256 MiB"),
                   ("c3", "C3: 512 MiB UTF-16LE")]:
    r = pc[cfg]
    for op in ["utf8_validate", "utf8_to_utf16le_planned", "utf16le_validate",
               "utf16le_to_utf8_planned"]:
        v = r[op]
        row(label, names[op], v["input_gbs"], v["gchar_per_s"], v["hbm_gbs"], par)
ch = c["chars"]
for op, key in [("UTF-8→UTF-16LE (two-pass)", "utf8_to_utf16le_planned"),
                ("UTF-16LE→UTF-8 (two-pass)", "utf16le_to_utf8_planned")]:
    v = po[key]
    row("C4: 8 GiB mixed", op, v["input_gbs"], ch / v["ms"] / 1e6, v["hbm_gbs"],
        "bit-exact on all 128 chunks, sharded G=2/4/8 equal, 16 error copies per G",
        f"{cb['single_thread']['value']:.2f}*", f"{cb['value']:.2f}* ({cb['cores']} threads)")
table = "\n".join(rows)
text = open("BASELINE.md").read()
head = text[:text.index("## 4. Measured results")]
new = f"""## 4. Measured results (round 2; `profiles/{tag}_bench_default.json`, one B200, {d['clocks']['sm_mhz']:.0f} MHz)

Per-GPU numbers at G = 1. The 8 GiB config-4 step (the bench line: two-pass sizing + transcode,
both directions) runs at **{d['value']:.1f} GB/s** of input ({c['gchar_per_s']:.0f} Gchar/s); end to end
through the host-buffer API {d['e2e']['value']:.1f} GB/s. The scaling curve at G = 2 / 4 / 8 is the
driver's (SCALE_rNN.json); nothing here was measured on more than one GPU. HBM TB/s counts input
read + output written (algorithmic bytes; ncu DRAM bytes of the two transcoders measured at 8 GiB
are 1.00× of it).

| Config | Op | G | Input GB/s per GPU | Gchar/s per GPU | HBM TB/s | % of 8 TB/s | % of 6.45 TB/s | Oracle 1-core GB/s | Oracle N-core GB/s | Parity |
|---|---|---|---|---|---|---|---|---|---|---|
{table}

\\* The oracle columns are the whole four-op step (len16 + UTF-8→UTF-16LE + len8 + UTF-16LE→UTF-8)
on 64 MiB chunks of config 4, input bytes of both transcoding passes per second: one thread
pinned to one core, and one thread per chunk on the box's cores. Validators and the C1–C3 ops
were not timed on the oracle separately.
"""
open("BASELINE.md", "w").write(head + new)
print("BASELINE.md section 4 from", tag)
