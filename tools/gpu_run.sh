# One parameterised GPU session (replaces the round-1 one-off scripts).  Usage on the box:
#   bash tools/gpu_run.sh TAG [STEP ...]
# STEP: tests[:<pytest -k expr>] | smoke | bench[:<bench.py args, commas for spaces>] | ref | launches[:args]
#       | ncufull:<kernel regex>:<bench.py args>| traffic:<kernel regex>:<args> | sanitize:<tool>:<pytest -k expr>
# Outputs land in gpurun_out/TAG_*.
set -u
TAG=$1; shift
mkdir -p gpurun_out
O=gpurun_out/$TAG
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > ${O}_smi.txt 2>&1
for STEP in "$@"; do
  KIND=${STEP%%:*}; ARG=""; [ "$KIND" != "$STEP" ] && ARG=${STEP#*:}
  case $KIND in
    tests)
      if [ -n "$ARG" ]; then timeout 2400 python -m pytest tests -m gpu -x -q -k "$ARG" > ${O}_pytest.log 2>&1
      else timeout 2400 python -m pytest tests -m gpu -x -q > ${O}_pytest.log 2>&1; fi
      echo "tests=$?"; tail -4 ${O}_pytest.log ;;
    smoke)
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > ${O}_smoke.log 2>&1; echo "smoke=$?"; tail -3 ${O}_smoke.log ;;
    bench)
      A=${ARG//,/ }; N=$(echo "$A" | tr -c 'a-z0-9' '_' | cut -c1-40)
      timeout 1200 python bench.py $A > ${O}_bench_${N}.log 2>&1; echo "bench[$A]=$?"
      tail -1 ${O}_bench_${N}.log | python tools/bench_brief.py ;;
    ref)
      timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > ${O}_bench_ref.log 2>&1; echo "ref=$?"; tail -c 600 ${O}_bench_ref.log ;;
    launches)
      A=${ARG//,/ }
      timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ${O}_launches.csv \
        python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e $A > ${O}_launches.log 2>&1; echo "launches=$?"
      python tools/ncu_summary.py --launches ${O}_launches.csv > ${O}_launches.txt 2>&1; head -20 ${O}_launches.txt ;;
    ncufull)
      RX=${ARG%%:*}; A=${ARG#*:}; A=${A//,/ }
      timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"$RX" -c 3 -o ${O}_full \
        python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e $A > ${O}_ncufull.log 2>&1; echo "ncufull=$?"
      tail -3 ${O}_ncufull.log
      python tools/ncu_summary.py ${O}_full.ncu-rep > ${O}_full.txt 2>&1; head -60 ${O}_full.txt ;;
    traffic)
      RX=${ARG%%:*}; A=${ARG#*:}; A=${A//,/ }
      timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
        -k regex:"$RX" --csv --log-file ${O}_traffic.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e $A \
        > ${O}_traffic.log 2>&1; echo "traffic=$?"; tail -20 ${O}_traffic.csv ;;
    sanitize)
      TOOL=${ARG%%:*}; K=${ARG#*:}
      timeout 2400 compute-sanitizer --tool $TOOL --print-limit 50 python -m pytest tests -m gpu -x -q -k "$K" \
        > ${O}_sanitize_${TOOL}.log 2>&1; echo "sanitize[$TOOL]=$?"; tail -8 ${O}_sanitize_${TOOL}.log ;;
  esac
done
