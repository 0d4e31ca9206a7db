"""Markdown table of a parity log (tests/gpu_util.py parity_log records, $BLSTM_PARITY_LOG): worst
per-tensor error per case and its margin to the path's tolerance (outputs normwise 1e-3, gradients
rel-L2 1e-2).  usage: python scripts/parity_table.py LOG.jsonl > OUT.md"""
import json
import sys

OUT_TOL, GRAD_TOL = 1e-3, 1e-2


def main():
    recs = [json.loads(l) for l in open(sys.argv[1]) if l.strip()]
    print(f"# Parity magnitudes (GPU vs fp64 oracle), from `{sys.argv[1].split('/')[-1]}`\n")
    print("Outputs: normwise max|g-r|/max|r| per tensor (tolerance 1e-3); gradients: rel-L2 per parameter "
          "tensor (tolerance 1e-2). precision 0 = BLSTM_PREC_FP16 (default), 1 = BLSTM_PREC_FP16X2W.\n")
    print("| Case | metric | tensors | tightest tensor | margin to its tolerance |")
    print("|---|---|---|---|---|")
    for r in recs:
        errs, metric = r["errors"], r.get("metric", "")

        def tol_of(name):
            if isinstance(metric, dict):  # {'y,c,hT,cT': 'normwise', 'rest': 'rel-L2'}
                outs = next((k for k, v in metric.items() if v == "normwise"), "").split(",")
                return OUT_TOL if name.split("[")[0] in outs else GRAD_TOL
            return OUT_TOL if metric == "normwise" else GRAD_TOL
        margins = {k: tol_of(k) / v if v > 0 else float("inf") for k, v in errs.items()}
        k = min(margins, key=margins.get)
        m = metric if isinstance(metric, str) else "outputs normwise, gradients rel-L2"
        print(f"| {r['case']} | {m} | {len(errs)} | {errs[k]:.2e} ({k}) | {margins[k]:.2f}x |")

if __name__ == "__main__":
    main()
