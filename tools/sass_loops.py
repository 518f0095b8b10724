"""List the innermost window loops of a kernel's SASS (cuobjdump -sass output
on stdin or as argv[1]): loop head, body size, LDS / POPC / local-memory
counts -- a quick check of what a code change did to the hot loop."""
import re
import sys

src = open(sys.argv[1]).read() if len(sys.argv) > 1 else sys.stdin.read()
ins = []
for line in src.split("\n"):
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr = {a: i for i, (a, _) in enumerate(ins)}
show = "-v" in sys.argv
for i, (a, t) in enumerate(ins):
    if "BRA" not in t:
        continue
    m = re.search(r"0x([0-9a-f]+)", t.split("BRA")[-1])
    if not m:
        continue
    ta = int(m.group(1), 16)
    if ta < a and ta in addr and i - addr[ta] < 400:
        body = ins[addr[ta]:i + 1]
        npc = sum("POPC" in x for _, x in body)
        if npc >= 7:
            print(hex(ta), len(body), "LDS", sum("LDS" in x for _, x in body), "POPC", npc,
                  "LDL/STL", sum(("LDL" in x or "STL" in x) for _, x in body))
            if show:
                for aa, tt in body:
                    print("   ", hex(aa), tt)
