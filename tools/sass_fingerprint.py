"""Dev tool: per-kernel SASS fingerprints of a built library, for refactors that must leave the
kept kernels' instruction streams unchanged (kernel-parameter offsets normalised).

python tools/sass_fingerprint.py <lib.so> > a.txt ; ... ; diff a.txt b.txt
"""
import hashlib, re, subprocess, sys

out = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
funcs, cur, lines = {}, None, []
for ln in out.splitlines():
    m = re.match(r"\s*Function : (\S+)", ln)
    if m:
        if cur:
            funcs[cur] = lines
        cur, lines = m.group(1), []
        continue
    if cur is None:
        continue
    ins = re.sub(r"/\*[0-9a-f]{4,}\*/", "", ln)
    ins = re.sub(r"/\* 0x[0-9a-f]+ \*/", "", ins)
    ins = re.sub(r"c\[0x0\]\[0x[0-9a-f]+\]", "c[0x0][P]", ins).strip()
    if ins:
        lines.append(ins)
if cur:
    funcs[cur] = lines
for name in sorted(funcs):
    print(hashlib.sha1("\n".join(funcs[name]).encode()).hexdigest()[:16], len(funcs[name]), name)
