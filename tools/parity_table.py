"""Format a GSR_PARITY_LOG jsonl (tests/gpu_helpers.assert_grad_parity) as the table of
profiles/<round>/parity_<round>.txt: python tools/parity_table.py log.jsonl [header-note]"""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1]) if l.strip()]
note = sys.argv[2] if len(sys.argv) > 2 else ""
print("# Element-wise gradient parity, GPU vs the stage-wise oracle (STAGE + running error bounds)" +
      (f", {note}" if note else ""))
print("# Command: GSR_PARITY_LOG=... python -m pytest tests/test_gpu_parity.py tests/test_gpu_keymask.py "
      "tests/test_gpu_naive.py -m gpu")
print("# Rule per element: |g - ref| <= max(1e-6 * scale, 1e-3 |ref|, C u M), C = 8, u = 2^-24,")
print("# M = the oracle's running error bound (oracle/gsref.cpp struct Rn, DESIGN.md §6).  No fraction allowance.")
print("#   worst/allowed : max over elements of |g - ref| / allowed   (must be <= 1)")
print("#   worst/uM      : max over elements of |g - ref| / (u M)     (C = 8 leaves this much headroom)")
print("#   >north_star   : elements outside 'rel 1e-3 or abs 1e-6' alone, each explained by the bound")
print("#   relaxed       : elements whose allowed error is the bound term (ill-conditioned sums)")
print("#   nonzero       : elements with a nonzero reference")
print(f"{'test':70s} {'what':8s} {'worst/allowed':>13s} {'worst/uM':>9s} {'>north_star':>11s} {'relaxed':>8s} "
      f"{'nonzero':>8s}")
for r in rows:
    t = r["test"].replace("tests/", "")
    print(f"{t:70s} {r['what'][:8]:8s} {r['worst_ratio']:13.3f} {r['worst_ratio_vs_u_M']:9.2f} "
          f"{r['outside_north_star_tol']:11d} {r['relaxed_by_bound']:8d} {r['nonzero_ref']:8d}")
print(f"# {len(rows)} checks, worst/allowed max {max(r['worst_ratio'] for r in rows):.3f}")
