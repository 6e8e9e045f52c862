"""List the loops (backward branches) of a cuobjdump -sass dump with their instruction mix."""
import re, sys, collections
lines = open(sys.argv[1]).read().splitlines()
ins = []
for l in lines:
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)\s*([^;]*);", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(3), m.group(4)))
addr = {a: i for i, (a, _, _) in enumerate(ins)}
for i, (a, op, args) in enumerate(ins):
    if op.startswith("BRA"):
        t = re.search(r"0x([0-9a-f]+)", args)
        if t and int(t.group(1), 16) < a:
            j = addr.get(int(t.group(1), 16))
            if j is None:
                continue
            body = ins[j:i + 1]
            c = collections.Counter(o.split(".")[0] for _, o, _ in body)
            print(f"loop 0x{int(t.group(1),16):x}-0x{a:x}: {len(body)} instr: " + ", ".join(f"{k} {v}" for k, v in c.most_common(14)))
