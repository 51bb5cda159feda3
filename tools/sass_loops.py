"""Tools only: list the loops (backward branches) of a cuobjdump -sass function dump with an
opcode histogram of each loop body.  usage: sass_loops.py file.sass [min_instructions]"""
import re, sys, collections
lines = open(sys.argv[1]).read().splitlines()
minlen = int(sys.argv[2]) if len(sys.argv) > 2 else 40
ins = []
for l in lines:
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr_index = {a: k for k, (a, _) in enumerate(ins)}
for k, (a, t) in enumerate(ins):
    m = re.search(r"\bBRA\S*\s+(?:\S+,\s*)?`?\(?\.?L?_?x?_?(\w+)\)?|BRA\S* (0x[0-9a-f]+)", t)
    m2 = re.search(r"BRA.*?0x([0-9a-f]+)", t)
    if "BRA" in t and m2:
        tgt = int(m2.group(1), 16)
        if tgt < a and tgt in addr_index:
            body = ins[addr_index[tgt]:k + 1]
            if len(body) < minlen:
                continue
            h = collections.Counter()
            for _, b in body:
                op = re.sub(r"^@!?U?P\d+\s+", "", b).split()[0]
                key = op.split(".")[0]
                if op.startswith("IMAD.MOV") or op.startswith("MOV"):
                    key = "MOV*"
                h[key] += 1
            print(f"loop {tgt:#x}..{a:#x}: {len(body)} instr  " + " ".join(f"{o}:{c}" for o, c in h.most_common(18)))
