"""Per-kernel SASS instruction counts of the built library (cuobjdump -sass):
the evidence that the hot kernels run on the FP64 tensor pipe (DMMA), the
5th-gen tensor cores (UTC*MMA + LDTM/STTM for TMEM) and the copy engines of
TMA / bulk copies (UTMALDG / UBLKCP).  usage: python tools/sass_summary.py [lib]"""
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2010_00465_b200/libcossin_b200.so"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True,
                      check=True).stdout
COLS = [("DMMA", r"\bDMMA\."), ("DFMA", r"\bDFMA\b"), ("UTC*MMA", r"\bUTC\w*MMA\b"),
        ("LDTM", r"\bLDTM\b"), ("STTM", r"\bSTTM\b"), ("UTMALDG", r"\bUTMALDG\b"),
        ("UBLKCP", r"\bUBLKCP\b"), ("LDGSTS", r"\bLDGSTS\b"), ("LDS", r"\bLDS\b"),
        ("SYNCS", r"\bSYNCS\b")]
rows, name, body = [], None, []


def flush():
    if name:
        text = "\n".join(body)
        total = sum(1 for l in body if re.search(r"/\*[0-9a-f]{4,}\*/", l))
        rows.append((name, total, [len(re.findall(p, text)) for _, p in COLS]))


for line in sass.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        flush()
        name, body = m.group(1), []
    elif name:
        body.append(line)
flush()
demangled = subprocess.run(["c++filt"], input="\n".join(r[0] for r in rows),
                           capture_output=True, text=True).stdout.splitlines()
print(f"# cuobjdump -sass {lib.split('/')[-1]} (sm_100a): per-kernel instruction counts")
print("# kernel | total | " + " | ".join(c for c, _ in COLS))
for (nm, total, cnt), dm in sorted(zip(rows, demangled), key=lambda x: -x[0][1]):
    dm = (re.sub(r"\(.*", "", dm) or nm)[:90]
    print(f"{dm} | {total} | " + " | ".join(str(c) for c in cnt))
