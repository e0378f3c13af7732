"""Static SASS instruction count per source line of k_fused_plan<1> (nvdisasm line info of a
-lineinfo cubin), for a line range of fused.cu.  Usage: sass_lines.py ALL.SASS FIRST LAST"""
import collections, re, sys

lines = open(sys.argv[1]).read().split("\n")
lo, hi = int(sys.argv[2]), int(sys.argv[3])
start = end = None
for i, l in enumerate(lines):
    if ".text._ZN2ss12k_fused_planILi1EEEvNS_9FusedArgsIXT_EEE:" in l:
        start = i
    elif start is not None and i > start and re.match(r"\s*\.text\.", l):
        end = i
        break
cur, cnt = None, collections.Counter()
for l in lines[start:end]:
    if "//## File" in l:
        m = re.search(r'"([^"]+)", line (\d+)', l)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    if re.search(r"/\*[0-9a-f]{4}\*/", l):
        cnt[cur] += 1
src = open("paper_2601_21473_b200/csrc/fused.cu").read().split("\n")
tot = 0
for k, v in sorted((k, v) for k, v in cnt.items() if k and k[0] == "fused.cu" and lo <= k[1] <= hi):
    tot += v
    print(k[1], v, src[k[1] - 1].strip()[:90])
print("static SASS in range", tot, "of", sum(cnt.values()))
