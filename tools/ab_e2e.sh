for rep in 1 2 3; do
  for lib in "" d2; do
    echo -n "rep $rep lib=${lib:-cur}: "; LSG_LIB=$lib python tools/pipe_trace.py cfg5 10 2>/dev/null
  done
done
./tools/duplex_probe | head -4
