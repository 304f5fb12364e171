"""Static SASS size of one kernel by source file:line (needs -lineinfo).

usage: python tools/sass_lines.py <lib.so> <mangled kernel name> [N]
"""
import collections
import os
import re
import subprocess
import sys
import tempfile


def main():
    lib, fn = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    out = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
    cnt, infn, cur = collections.Counter(), False, None
    for line in out.splitlines():
        if ".section\t.text." in line:
            infn = line.split(".text.")[1].split(",")[0] == fn
            continue
        if not infn:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', line)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        if re.match(r"\s+/\*[0-9a-f]{4,}\*/", line):
            cnt[cur] += 1
    tot = sum(cnt.values())
    byf = collections.Counter()
    for k, c in cnt.items():
        byf[k[0] if k else None] += c
    print(f"{fn}: {tot} instructions ({tot * 16 // 1024} KB)")
    print({k: v for k, v in byf.most_common()})
    for k, c in cnt.most_common(top):
        print(c, k)


if __name__ == "__main__":
    main()
