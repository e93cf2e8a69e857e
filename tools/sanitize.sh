#!/bin/bash
# compute-sanitizer evidence: memcheck over the smoke step (fp32 + bf16 DASH step:
# sampling, advantage, accumulate, Adam) and a few GPU parity tests (tcgen05 GEMMs, attention,
# paged decode with retirement, PPO / KL, the fused optimizer), synccheck over the smoke step.
# Run on the GPU box from the repo root; summaries land in gpurun_out/sanitize_*.log.
set -u
O=gpurun_out
mkdir -p $O
CS="compute-sanitizer --print-limit 20 --error-exitcode 9"
timeout 1200 $CS --tool memcheck python -c "import __graft_entry__ as g; g.smoke()" > $O/sanitize_memcheck_smoke.log 2>&1
echo "memcheck smoke rc=$?" >> $O/sanitize_summary.log
timeout 1200 $CS --tool synccheck python -c "import __graft_entry__ as g; g.smoke()" > $O/sanitize_synccheck_smoke.log 2>&1
echo "synccheck smoke rc=$?" >> $O/sanitize_summary.log
timeout 2400 $CS --tool memcheck python -m pytest tests -m gpu -q -x \
  -k "bit_exact_under_logits_dump and qwenlike or retirement or fused_step_virtual or ppo_at_entry or kl_term_vs or long_sequences_hd128 or tc_gemm_epilogues" \
  > $O/sanitize_memcheck_tests.log 2>&1
echo "memcheck tests rc=$?" >> $O/sanitize_summary.log
tail -3 $O/sanitize_memcheck_smoke.log $O/sanitize_synccheck_smoke.log $O/sanitize_memcheck_tests.log >> $O/sanitize_summary.log
