"""Regenerate the committed SASS evidence from the built libmhg.so:
  profiles/TAG_sass_census.txt     opcode census (tcgen05 / TMA / mbarrier) per GEMM kernel
  profiles/TAG_sass_k_gemm_L2.txt  trimmed listing of the headline kernel k_gemm<2, fold 2>
(python profiles/sass_evidence.py [TAG], TAG defaults to r02)
tcgen05.mma -> UTCIMMA (kind::i8), tcgen05.ld -> LDTM, tcgen05.commit -> UTCBAR,
cp.async.bulk -> UBLKCP, cp.async.bulk.tensor -> UTMALDG, mbarrier -> SYNCS.*"""
import collections
import os
import re
import subprocess
import sys

here = os.path.dirname(os.path.abspath(__file__))
TAG = sys.argv[1] if len(sys.argv) > 1 else "r02"
lib = os.path.join(os.path.dirname(here), "paper_1705_04807_b200", "libmhg.so")
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs, cur = {}, None
for line in sass.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = []
    elif cur:
        funcs[cur].append(line)
KEYS = ("UTCIMMA", "UTCBAR", "LDTM", "UBLKCP", "UTMALDG", "SYNCS", "UTCATOMSWS", "STTM")
out = ["# SASS opcode census of libmhg.so (cuobjdump -sass), per GEMM kernel",
       "# " + __doc__.splitlines()[3]]
for name in sorted(funcs):
    if "k_gemm" not in name:
        continue
    short = re.search(r"(k_gemm2?I[^E]*E(?:Li\d+E)?(?:Lb\d)?)", name)
    cnt = collections.Counter()
    ninstr = 0
    for line in funcs[name]:
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Za-z0-9_.]+)", line)
        if m:
            ninstr += 1
            op = m.group(1)
            if op.startswith(KEYS):
                cnt[op] += 1
    out.append(f"== {short.group(1) if short else name[:60]} ({ninstr} instructions) {name}")
    for op, c in cnt.most_common():
        out.append(f"  {c:5d} {op}")
open(os.path.join(here, f"{TAG}_sass_census.txt"), "w").write("\n".join(out) + "\n")

target = [n for n in funcs if re.search(r"k_gemmILi2ELi2EE", n)]
lines = funcs[target[0]] if target else []
keep = set()
for i, line in enumerate(lines):
    if re.search(r"UTCIMMA|UTCBAR|UBLKCP|LDTM|SYNCS\.ARRIVE", line):
        keep.update(range(max(0, i - 6), min(len(lines), i + 7)))
lst = [f"# {target[0] if target else 'k_gemm<2,2>'} SASS (cuobjdump -sass libmhg.so), trimmed to the",
       "# tcgen05 / bulk-copy / TMEM regions: MMA issue (UTCIMMA), commits (UTCBAR), bulk copies",
       f"# (UBLKCP), TMEM loads (LDTM), mbarrier arrives, +-6 lines of context; full function: {len(lines)} lines"]
prev = -2
for i in sorted(keep):
    if i != prev + 1:
        lst.append("        ...")
    lst.append(re.sub(r"\s*/\* 0x[0-9a-f]+ \*/\s*$", "", lines[i]))
    prev = i
open(os.path.join(here, f"{TAG}_sass_k_gemm_L2.txt"), "w").write("\n".join(lst) + "\n")
print("\n".join(out[:40]))
