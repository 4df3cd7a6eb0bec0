"""List reference citations (file.py:N[-M]) that point past the end of the
cited reference file.  Run in the build container (reads /root/reference)."""
import os
import re
import sys

REF = "/root/reference/pkg/src/conesplit"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lens = {f: sum(1 for _ in open(os.path.join(REF, f))) for f in os.listdir(REF) if f.endswith(".py")}
for extra in ("SPEC.md", "PAPER.md"):
    for base in ("/root/reference", "/root/reference/pkg"):
        p = os.path.join(base, extra)
        if os.path.exists(p):
            lens[extra] = sum(1 for _ in open(p))
pat = re.compile(r"\b(" + "|".join(re.escape(f) for f in lens) + r"):(\d+)(?:-(\d+))?((?:,\s*:\d+(?:-\d+)?)*)")
bad = 0
for dp, dn, fn in os.walk(ROOT):
    if any(x in dp for x in (".git", "golden", "gpurun_out", "__pycache__", "profiles")):
        continue
    for f in fn:
        if not f.endswith((".py", ".cu", ".cuh", ".h", ".cpp", ".md")) or f in ("SURVEY.md", "VERDICT.md", "BASELINE.md", "PAPERS.md", "SNIPPETS.md", "ADVICE.md"):
            continue
        path = os.path.join(dp, f)
        for i, line in enumerate(open(path, errors="replace"), 1):
            for m in pat.finditer(line):
                ref, a, b, rest = m.group(1), int(m.group(2)), m.group(3), m.group(4)
                nums = [a] + ([int(b)] if b else []) + [int(x) for x in re.findall(r"\d+", rest or "")]
                if max(nums) > lens[ref]:
                    bad += 1
                    print(f"{os.path.relpath(path, ROOT)}:{i}: {m.group(0)}  (len {lens[ref]})")
print(f"{bad} out-of-range citations", file=sys.stderr)
