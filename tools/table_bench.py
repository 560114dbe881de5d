"""The reference's bench mode (src/cli.py:233-252) through this package: constant-time
scaling sweep of VoxelTable accumulate_batch + lookup_slots, 1e5 .. 1e7 vertices with
proportional capacity (SPEC criterion 6).  usage: python tools/table_bench.py [--json f]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1902_05942_b200 import bench  # noqa: E402


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--json", default=None)
    ap.add_argument("--repeats", type=int, default=3)
    args = ap.parse_args()
    bench.run_point(100_000)  # first call: module and kernel loading
    out = {}
    for mode in ("fixed", "float"):
        pts = bench.scaling_sweep((100_000, 1_000_000, 10_000_000), sum_mode=mode,
                                  repeats=args.repeats)
        for p in pts:
            print(f"sum_mode={mode} {p.line()}")
        print(f"sum_mode={mode} per_vertex_spread={bench.spread(pts):.3f} "
              f"device_per_vertex_spread={bench.spread(pts, device=True):.3f}")
        out[mode] = {"points": [dict(n=p.n_vertices, capacity=p.capacity,
                                     accumulate_s=p.accumulate_s, lookup_s=p.lookup_s,
                                     per_vertex_ns=p.per_vertex_ns, device_s=p.device_s,
                                     device_per_vertex_ns=p.device_per_vertex_ns)
                                for p in pts],
                     "per_vertex_spread": bench.spread(pts),
                     "device_per_vertex_spread": bench.spread(pts, device=True)}
    if args.json:
        with open(args.json, "w") as f:
            json.dump(out, f, indent=1)
    return 0


if __name__ == "__main__":
    sys.exit(main())
