"""Per-kernel registers / spills from `nvcc -Xptxas -v` output (stdin or a log file)."""
import re
import subprocess
import sys

text = open(sys.argv[1]).read() if len(sys.argv) > 1 else sys.stdin.read()
cur = None
rows = {}
for line in text.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        rows[cur] = {}
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and "spill" not in rows[cur]:
        rows[cur]["spill"] = (int(m.group(1)), int(m.group(2)))
    m = re.search(r"Used (\d+) registers", line)
    if m:
        rows[cur]["regs"] = int(m.group(1))
names = list(rows)
try:
    dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True,
                         text=True).stdout.splitlines()
except OSError:
    dem = names
for n, d in zip(names, dem):
    r = rows[n]
    sp = r.get("spill", (0, 0))
    flag = "  SPILL" if sp[0] or sp[1] else ""
    print(f"{r.get('regs', '?'):>4} regs  spill {sp[0]:>4}/{sp[1]:<4} {d[:110]}{flag}")
