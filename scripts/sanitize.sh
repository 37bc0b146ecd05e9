# compute-sanitizer evidence: racecheck, synccheck, memcheck and
# initcheck over one small launch of every kernel family
# (scripts/sanitize_cases.py, oracle-checked).  Summaries land in
# gpurun_out/$TAG.sanitize.<tool>.log; profiles/ keeps the committed copy.
# Usage (via gpurun): bash scripts/sanitize.sh TAG
TAG=${1:-san}
mkdir -p gpurun_out
python -c "import paper_2306_16731_b200 as f; f.load_library()"  # page the image in outside the tools
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  log=gpurun_out/$TAG.sanitize.$tool.log
  echo "== $tool" > $log
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 20 \
      python scripts/sanitize_cases.py >> $log 2>&1
  echo "rc=$?" >> $log
  grep -E "CASE|ERROR SUMMARY|RACECHECK SUMMARY|Error|error|rc=" $log | tail -40
done
