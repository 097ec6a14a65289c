#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/step_timeline.py c2 20 10 gpurun_out/timeline_c2.json > gpurun_out/timeline_c2.log 2>&1
echo "tl rc=$?"; grep -v Warn gpurun_out/timeline_c2.log | grep -v "^  .* us  x" | head -n 20
SF_GMRES_GRAPH=1 timeout 600 python tools/step_timeline.py c2 20 10 gpurun_out/timeline_c2_graph.json > gpurun_out/timeline_c2_graph.log 2>&1
echo "tlg rc=$?"; grep -v Warn gpurun_out/timeline_c2_graph.log | grep -v "^  .* us  x" | head -n 20
timeout 600 python tools/step_timeline.py c3_scaled 3 3 gpurun_out/timeline_c3s.json > gpurun_out/timeline_c3s.log 2>&1
echo "tl3 rc=$?"; grep -v Warn gpurun_out/timeline_c3s.log | head -n 16
