# usage: bash tools/build_variants.sh name1:"-DFLAG ..." name2:"..."   -> tools/variants/<name>.so
set -e
rm -rf tools/variants; mkdir -p tools/variants
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  VT_NVCC_EXTRA="$flags" python -m paper_2109_10433_b200.build --force > /dev/null
  cp paper_2109_10433_b200/lib/libvtrans_gpu.so tools/variants/$name.so
  echo "$name: $flags $(grep -A2 'utf8_transcode_kernelILb0' paper_2109_10433_b200/lib/ptxas.log | grep -o 'Used [0-9]* registers\|[0-9]* bytes spill stores' | tr '\n' ' ')"
done
python -m paper_2109_10433_b200.build --force > /dev/null
