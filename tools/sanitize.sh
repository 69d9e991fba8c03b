#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over the small
# production cases; plain stream launches (CMG_NO_GRAPH=1) plus one memcheck
# pass through the CUDA-graph path.  Logs -> gpurun_out/$1/
O=gpurun_out/${1:-sanitizer}; mkdir -p $O
export CMG_NO_GRAPH=1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_case.py > $O/$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $O/$tool.log | tail -1)"
done
unset CMG_NO_GRAPH
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_case.py > $O/memcheck_graph.log 2>&1
echo "memcheck (graph) rc=$? $(grep -E 'ERROR SUMMARY' $O/memcheck_graph.log | tail -1)"
