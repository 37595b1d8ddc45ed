# r03s: ncu captures of the hot kernels, summarised on the box (the reps plus the launch lists exceed the merge cap)
O=gpurun_out; mkdir -p $O; T=r03r
sed -n '/^# the bench step/,$p' tools/profile_round.sh | grep -v k_gather_h | grep -v k_qfit | sed "s/\$TAG/$T/g; s/\$O/$O/g" > /tmp/caps.sh
bash /tmp/caps.sh
python tools/summarize_ncu.py $O/r03r_ncu_summary_b.md $O/ncu_{eval4,escatter,sweepw,prune}_$T.ncu-rep
ls -la $O
