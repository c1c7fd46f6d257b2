"""Summarises bench.py JSON lines (one file per line) into the markdown table kept under profiles/.

usage: python profiles/bench_lines.py out.md line1.json [line2.json ...]
"""
import json
import sys


def row(path):
    d = json.loads(open(path).read().strip().splitlines()[-1])
    r = d.get("roofline") or {}
    e2e = (d.get("e2e") or {}).get("value")
    cpu = d.get("cpu_baseline") or {}
    clk = d.get("clocks") or {}
    res = d.get("result") or {}
    return (f"| {d['config']['workload'][:60]} | {d['ms_per_step']:.3f} | {d['value']:.4g} | "
            f"{(e2e or 0):.4g} | {r.get('kernel', '')[:40]} | {r.get('frac', 0):.3f} | "
            f"{r.get('avg_launch_ms', 0):.3f} | {(r.get('share_of_step') or 0):.2f} | "
            f"{cpu.get('value') if cpu.get('value') is None else format(cpu['value'], '.3g')} ({cpu.get('cores')} cores) | "
            f"{clk.get('sm_mhz')} {','.join(clk.get('reasons', []))} | {json.dumps(res)[:80]} |"), d


def main():
    out, paths = sys.argv[1], sys.argv[2:]
    lines = ["| workload | ms/step | estimates/s | e2e | dominant kernel | roofline frac | ms/launch | share | "
             "CPU port (est/s) | SM MHz / reasons | result |", "|---|---|---|---|---|---|---|---|---|---|---|"]
    raw = []
    for p in paths:
        try:
            r, d = row(p)
            lines.append(r)
            raw.append(d)
        except Exception as exc:  # noqa: BLE001
            lines.append(f"| {p}: unreadable ({exc}) |")
    body = "\n".join(lines) + "\n\nRaw lines:\n\n```\n" + "\n".join(json.dumps(d) for d in raw) + "\n```\n"
    open(out, "w").write(body)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
