"""Human-readable table of a bench line's extra.shard_emulation.

    python tools/emulation_table.py profiles/r2_bench_c5.json
"""
import json
import sys


def main():
    text = open(sys.argv[1]).read().strip()
    d = json.loads(text) if text.startswith("{") and "\n" not in text.strip()[:2] else json.loads(text)
    em = d["extra"]["shard_emulation"]
    print(f"workload: {d['config']['workload']}")
    print(f"one-GPU step (graph replay, memset + K1 + K2): "
          f"{em['one_gpu_step_ms']:.4f} ms")
    print(f"method: {em['method']}")
    print()
    print(f"{'P':>2s} {'max shard ms':>13s} {'min shard ms':>13s} "
          f"{'tail ms':>8s} {'step ms':>8s} {'Tconf/s':>8s} {'eff':>6s} "
          f"{'tables':>7s}")
    for p in (2, 4, 8):
        e = em[f"P{p}"]
        print(f"{p:2d} {e['max_shard_ms']:13.4f} {e['min_shard_ms']:13.4f} "
              f"{e['tail_ms']:8.4f} {e['projected_step_ms']:8.4f} "
              f"{e['projected_configs_per_s'] / 1e12:8.2f} "
              f"{e['projected_efficiency']:6.3f} "
              f"{'exact' if e['combined_tables_exact'] else 'WRONG':>7s}")
    print()
    for p in (2, 4, 8):
        e = em[f"P{p}"]
        print(f"P{p} shards (ms): " + " ".join(f"{x:.4f}" for x in e["shard_ms"]))
        if "shard_plans" in e:
            print("   model wavefronts/RED: " + " ".join(
                f"{pl['model_wavefronts_per_red']:.4f}" for pl in e["shard_plans"]))
        if "multi_entry_shard_ms" in e:
            print("   via isd_enumerate_multi (one call, events per shard): " +
                  " ".join(f"{x:.4f}" for x in e["multi_entry_shard_ms"]))


if __name__ == "__main__":
    main()
