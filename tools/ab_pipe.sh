# lsg_solver_step_host upload plans on cfg5 512^3 (same box, interleaved), then one
# traced step of the default plan:  gpurun -- bash tools/ab_pipe.sh
for rep in 1 2; do
  for order in 1 0; do
    echo -n "rep $rep LSG_PIPE_ORDER=$order: "; LSG_PIPE_ORDER=$order python tools/pipe_trace.py cfg5 10 2>/dev/null
  done
done
LSG_PIPE_TRACE=1 python tools/pipe_trace.py cfg5 3 2>&1 | tail -60
