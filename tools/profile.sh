# usage: bash tools/profile.sh <tag> <kernel-regex> <bench args...>
# Plain run first (must exit 0), then the launch list and one --set full capture.
mkdir -p gpurun_out
tag=$1; kre=$2; shift 2
python bench.py "$@" > gpurun_out/${tag}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/${tag}_launches.csv python bench.py "$@" > gpurun_out/${tag}_ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${kre} -s 4 -c 1 \
    -o gpurun_out/${tag} python bench.py "$@" > gpurun_out/${tag}_ncu2.log 2>&1
echo profile_rc=$?
tail -3 gpurun_out/${tag}_plain.log | cut -c1-300
