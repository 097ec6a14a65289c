"""Per-function SASS opcode histogram of a cubin/.so (cuobjdump -sass)."""
import collections
import re
import subprocess
import sys


def functions(path):
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    cur, body = None, []
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            if cur:
                yield cur, body
            cur, body = m.group(1), []
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if m and cur:
            body.append(m.group(2))
    if cur:
        yield cur, body


if __name__ == "__main__":
    path, pat = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    for name, body in functions(path):
        if pat in name:
            c = collections.Counter(op.split(".")[0] for op in body)
            print(name, len(body))
            print("  ", ", ".join(f"{k}:{v}" for k, v in c.most_common(30)))
