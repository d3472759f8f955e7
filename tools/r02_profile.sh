#!/bin/bash
# Round-2 measurement evidence (run under gpurun): launch lists of one eager
# step (C3, C2, C4 EGNN), ncu --set full of the C3 aggregation kernels and
# the C3 weight-gradient GEMM.  Each ncu command runs only after the same
# command exited 0 without ncu.
mkdir -p gpurun_out
for c in c3 c2 c4; do
  python tools/step_once.py --config $c --steps 1 > gpurun_out/plain_$c.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_$c.csv python tools/step_once.py --config $c --steps 1 \
      > gpurun_out/ncu_launch_$c.log 2>&1
  python tools/share.py gpurun_out/launches_$c.csv 1 > gpurun_out/share_$c.txt 2>&1
done
tools/ncu_one.sh c3 aggbwd "k_agg_bwd_vec" 0
tools/ncu_one.sh c3 aggfwd "k_agg_fwd_vec" 0
# the third flushed weight-gradient launch of the step = layer 5's [dW | dU | db]
tools/ncu_one.sh c3 wgrad "tc_gemm_tma_kernel<\(int\)128, gfm::tc::TcEpiPartial, \(int\)2, \(bool\)1>" 2
for t in aggbwd aggfwd wgrad; do echo "== $t"; cat gpurun_out/one_$t.txt; done
cat gpurun_out/share_c3.txt gpurun_out/share_c2.txt gpurun_out/share_c4.txt
