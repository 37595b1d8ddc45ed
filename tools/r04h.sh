#!/bin/bash
# r04h: build chain timeline (device events vs host returns), engine trace
O=gpurun_out; mkdir -p $O
timeout 300 python tools/probe_build_timeline.py > $O/r04h_timeline.log 2>&1
WT_TRACE_ENGINE=1 timeout 300 python tools/probe_build_timeline.py > $O/r04h_timeline_trace.log 2>&1
WT_FIT_TRACE=2 timeout 300 python tools/probe_build_timeline.py > $O/r04h_timeline_fit.log 2>&1
