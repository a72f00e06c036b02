"""Dev tool: markdown table of tools/sweep.py JSON lines.  usage: python tools/sweep_table.py FILE..."""
import json
import sys

print("| GPUs | tokens | experts | PPMoE tokens/s | all-to-all tokens/s | PPMoE / a2a |")
print("|---|---|---|---|---|---|")
for f in sys.argv[1:]:
    for line in open(f):
        line = line.strip()
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        print(f"| {d['n_gpus']} | {d['tokens']} | {d['experts']} | {d['ppmoe_tok_s']:,.0f} | "
              f"{d['a2a_tok_s']:,.0f} | {d['ppmoe_tok_s'] / d['a2a_tok_s']:.2f} |")
