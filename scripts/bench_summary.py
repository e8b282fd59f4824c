"""Print the key fields of bench.py JSON lines read from stdin (one per line)."""
import json
import sys

for line in sys.stdin:
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    if "impl" in d:
        print("reference", d.get("value"), d.get("cpu_baseline", {}).get("sample"))
        continue
    rf = d["roofline"]
    if "avg_launch_us" not in rf:                    # the one-CTA path: no HBM pass
        print(f'{d["config"]["m"]}x{d["config"]["n"]} N={d["n_gpus"]}: {d["value"]:.1f} piv/s  solve {d["ms_per_step"] * 1e3:.1f} us  '
              f'e2e {d["e2e"]["value"]:.1f}  cpu {d.get("cpu_baseline", {}).get("value")}  parity {d["parity"]}')
        continue
    print(f'{d["config"]["m"]}x{d["config"]["n"]} N={d["n_gpus"]}: {d["value"]:.1f} piv/s  solve {d["ms_per_step"]:.1f} ms  '
          f'upd {rf["avg_launch_us"]:.1f} us {rf["achieved"]:.0f} GB/s frac {rf["frac"]:.3f}  share {rf["update_share_of_loop"]:.3f}  '
          f'e2e {d["e2e"]["value"]:.1f}  launches {d["gpu_launches"]}  clocks {d["clocks"]}  parity {d["parity"]}')
