#!/bin/bash
# One GPU session: build, pytest -m gpu (optionally -k), then extra commands from $EXTRA (one per line).
# Usage: TAG=x PYTEST_K="expr" bash scripts/gpu_session.sh [cmdfile]  (cmdfile: one extra command per line)
tag=${TAG:-s}; out=gpurun_out/$tag; mkdir -p $out
free -g > $out/free.txt 2>&1; nproc >> $out/free.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $out/nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail -30 $out/build.log; exit 1; }
if [ "${PYTEST:-1}" = "1" ]; then
  timeout ${PYTEST_TIMEOUT:-1800} python -m pytest ${PYTEST_PATHS:-tests} -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} ${PYTEST_ARGS} > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
  tail -15 $out/pytest_gpu.log
fi
i=0
while IFS= read -r cmd; do
  [ -z "$cmd" ] && continue
  i=$((i+1)); echo "== [$i] $cmd"
  bash -c "$cmd" > $out/extra_$i.log 2>&1; echo "rc=$?"; tail -${EXTRA_TAIL:-3} $out/extra_$i.log
done < "${1:-/dev/null}"
