"""List reference citations (file.py:N or file.py:N-M) that point past the end
of the cited reference file.  Run here (the reference is not on the GPU box).

    python tools/check_citations.py
"""
import re
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
REF = Path("/root/reference/pkg/src/sqf2k")
REF_TESTS = Path("/root/reference/pkg/tests")
lengths = {p.name: len(p.read_text().splitlines()) for p in REF.glob("*.py")}
tlengths = {p.name: len(p.read_text().splitlines()) for p in REF_TESTS.glob("*.py")} if REF_TESTS.exists() else {}
pat = re.compile(r"\b([a-z_]+\.py):(\d+)(?:-(\d+))?")
bad = 0
for f in list(ROOT.rglob("*.py")) + list(ROOT.rglob("*.cu")) + list(ROOT.rglob("*.cuh")) + \
        list(ROOT.rglob("*.h")) + list(ROOT.rglob("*.c")) + list(ROOT.rglob("*.md")):
    if any(x in f.parts for x in ("gpurun_out", ".git", "_ref")) or f.name in ("SURVEY.md", "VERDICT.md", "ADVICE.md", "PAPERS.md", "SNIPPETS.md", "BASELINE.md"):
        continue
    for i, line in enumerate(f.read_text(errors="replace").splitlines(), 1):
        for m in pat.finditer(line):
            name, a, b = m.group(1), int(m.group(2)), int(m.group(3) or m.group(2))
            n = lengths.get(name) or tlengths.get(name)
            if n is None:
                continue
            if b > n or a > b or a < 1:
                bad += 1
                print(f"{f.relative_to(ROOT)}:{i}: {m.group(0)} (file has {n} lines)")
print(f"{bad} out-of-range citations", file=sys.stderr)
