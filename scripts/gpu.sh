#!/bin/bash
# One parameterised GPU-box runner (used as: gpurun -- bash scripts/gpu.sh <step> [<step> ...]).
# Steps: test | smoke | bench[:C] | ref[:C] | launches[:C] | ncu:<C>:<kernel-regex>:<skip>:<count>
# Logs go to gpurun_out/<tag>_<step>.log; TAG (env) prefixes them.
TAG=${TAG:-run}
mkdir -p gpurun_out
for step in "$@"; do
  IFS=: read -r what a b c d <<< "$step"
  log="gpurun_out/${TAG}_${what}${a:+_$a}.log"
  case "$what" in
    test)   timeout 1500 python -m pytest tests -m gpu -x -q --timeout 600 --timeout-method thread > "$log" 2>&1 ;;
    testk)  timeout 1500 python -m pytest tests -m gpu -q --timeout 600 --timeout-method thread -k "$a" > "$log" 2>&1 ;;
    bench1) timeout 900 python bench.py --only --no-cpu ${a:+--config $a} > "$log" 2>&1 ;;
    smoke)  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$log" 2>&1 ;;
    smokencu) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$log.plain" 2>&1 && \
            timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
              --log-file "gpurun_out/${TAG}_smoke_launches.csv" python -c "import __graft_entry__ as g; g.smoke()" > "$log" 2>&1 ;;
    benchall) timeout 1500 python bench.py > "$log" 2>&1 ;;
    bench)  timeout 900 python bench.py ${a:+--config $a} > "$log" 2>&1 ;;
    ref)    timeout 900 python bench.py --impl reference ${a:+--config $a} > "$log" 2>&1 ;;
    launches) timeout 300 python bench.py ${a:+--config $a} --no-cpu --steps 5 --warmup 3 > "$log.plain" 2>&1 && \
            RAC_PROFILE_NONCOOP=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
              --log-file "gpurun_out/${TAG}_launches_cfg${a}.csv" python bench.py ${a:+--config $a} --no-cpu --steps 5 --warmup 3 > "$log" 2>&1 ;;
    ncu)    timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$b" -s "${c:-0}" -c "${d:-1}" \
              -o "gpurun_out/${TAG}_ncu_cfg${a}" -f python scripts/prof_en.py "$a" 2 > "$log" 2>&1 ;;
    *)      echo "unknown step $step"; continue ;;
  esac
  echo "$step rc=$?"
done
