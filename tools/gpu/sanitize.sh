# usage (under gpurun): bash tools/gpu/sanitize.sh [tools...]   (default: racecheck synccheck memcheck)
# compute-sanitizer over tools/sanitize_run.py (every launch shape of the product path,
# including the in-launch update-pass CTAs that spin on the tail-completion counter).
mkdir -p gpurun_out
TOOLS=${*:-racecheck synccheck memcheck}
timeout 300 python tools/sanitize_run.py 64 > gpurun_out/sanitize_plain.log 2>&1; echo "plain rc=$?" >> gpurun_out/sanitize_plain.log
for t in $TOOLS; do
  extra=""
  [ "$t" = "racecheck" ] && extra="--racecheck-report all"
  timeout 1500 compute-sanitizer --tool $t $extra --print-limit 50 python tools/sanitize_run.py 64 \
      > gpurun_out/sanitize_$t.log 2>&1
  echo "$t rc=$?" >> gpurun_out/sanitize_$t.log
done
