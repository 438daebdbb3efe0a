# compute-sanitizer over every kernel (tools/sanitize.py), one tool at a time
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2c
python tools/sanitize.py > gpurun_out/r2c/plain.txt 2>&1; echo rc=$? >> gpurun_out/r2c/plain.txt
for t in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize.py > gpurun_out/r2c/$t.txt 2>&1
  echo "rc=$?" >> gpurun_out/r2c/$t.txt
done
