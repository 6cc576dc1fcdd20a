import re, sys
cur = ""
for line in open(sys.argv[1]):
    if line.startswith('=='):
        cur = line.strip()[3:]
        continue
    m = re.search(r"(\S+) -> (\S+)\s+\{.*'tile_records': (\d+), 'smem_bytes': (\d+).*'tma': (\w+).*\} ([\d.]+) ms (\d+) GB/s", line)
    if m:
        print(f"{cur:40s} {m.group(1):>8}->{m.group(2):<8} T={m.group(3):>5} smem={m.group(4):>6} {m.group(7)}")
    elif line.strip():
        print(line.strip()[:200])
