# lsg_solver_step_host variants on cfg5 512^3 (same box, interleaved), then one
# traced step of the default:  gpurun -- bash tools/ab_pipe.sh
for rep in 1 2; do
  for v in "LSG_PIPE_D2H_MIN=0" "LSG_PIPE_D2H_MIN=67108864" "LSG_PIPE_D2H_MIN=134217728" \
           "LSG_PIPE_D2H_MIN=268435456" "LSG_PIPE_K=24 LSG_PIPE_D2H_MIN=67108864" "LSG_PIPE_K=48"; do
    echo -n "rep $rep $v: "; env $v python tools/pipe_trace.py cfg5 10 2>/dev/null
  done
done
LSG_PIPE_TRACE=1 python tools/pipe_trace.py cfg5 3 2>&1 | tail -100
