"""Development tool: annotate cuobjdump -sass output with the control bits
(stall, yield, write/read scoreboard, wait mask) decoded from each
instruction's upper 64 bits.  Usage: sass_ctrl.py file.sass [start] [end]."""
import re
import sys

lines = open(sys.argv[1]).read().splitlines()
lo = int(sys.argv[2]) if len(sys.argv) > 2 else 0
hi = int(sys.argv[3]) if len(sys.argv) > 3 else len(lines)
ins = re.compile(r"/\*([0-9a-f]{4,})\*/\s+(.*?);?\s*/\* (0x[0-9a-f]+) \*/")
hexonly = re.compile(r"^\s*/\* (0x[0-9a-f]+) \*/\s*$")
i = lo
while i < min(hi, len(lines)):
    m = ins.search(lines[i])
    if m and i + 1 < len(lines):
        h = hexonly.match(lines[i + 1])
        if h:
            w = int(h.group(1), 16)
            stall = (w >> 41) & 0xF
            yld = (w >> 45) & 1
            wb = (w >> 46) & 7
            rb = (w >> 49) & 7
            wm = (w >> 52) & 0x3F
            wait = ",".join(str(b) for b in range(6) if wm >> b & 1)
            print(f"{i:6d} {m.group(1)} S{stall:2d}{'Y' if yld else ' '} W{wb if wb != 7 else '-'} R{rb if rb != 7 else '-'} "
                  f"wait[{wait:11s}] {m.group(2).strip()}")
            i += 2
            continue
    i += 1
