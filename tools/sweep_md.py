"""Development tool: render bench.py sweep lines (JSON, one per line) as the markdown table kept under
profiles/:  python tools/sweep_md.py profiles/round2_sweep.jsonl "round2 sweep" > profiles/round2_sweep.md"""
import json
import sys


def main():
    path, title = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "sweep"
    print(f"# {title} (bench.py lines, one B200, {path})\n")
    print("Each line: `python bench.py --no-cpu-baseline --no-e2e --steps 100 [...]` (ring of independent "
          "layer/X/Y sets so codes come from HBM; decode sizes replay CUDA graphs). Per-kernel times come from "
          "the eager profiled pass after the timed region (kernels serialised, no PDL overlap). `frac` = the "
          "dispatched kernel's roofline fraction (tensor: dense TFLOP/s of burst 1664.7; HBM: GB/s of 6556); "
          "`step` = the whole step against both roofs (time_lb / measured).\n")
    print("| shape (out x in) | T | bits (realized) | router h | µs/step | M tokens/s | router / gather / GEMM µs "
          "| GEMM kernel | kernel frac | step frac |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for line in open(path):
        line = line.strip()
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        c, k, r = d["config"], d.get("kernels", {}), d["roofline"]

        def us(name):
            v = k.get(name, {}).get("ms_per_launch", 0.0)
            return f"{v * 1e3:.1f}" if v else "-"
        print(f"| {c['out']}x{c['in']} | {c['tokens_per_step']} | {c['target_bits']} ({c['realized_avg_bits']}) "
              f"| {c['router_hidden']} | {d['ms_per_step'] * 1e3:.1f} | {d['value'] / 1e6:.3f} "
              f"| {us('router')} / {us('gather')} / {us('gemm')} | {c['kernels']['gemm']} | {r['frac']:.3f} "
              f"| {r['step'].get('achieved', r['step'].get('frac', 0.0)):.3f} |")


if __name__ == "__main__":
    main()
