# A/B of the working-tree library against HEAD's (_lib/variants/head.so) on
# K2 alone and the whole solve, then the GPU suite on the working tree.
set -x
mkdir -p gpurun_out
for cfg in cfg4 cfg2 cfg1; do
  for lib in head main; do
    if [ $lib = head ]; then export RKMF_LIB_PATH=$PWD/paper_2503_22631_b200/_lib/variants/head.so; else unset RKMF_LIB_PATH; fi
    timeout 300 python tools/kbench.py $cfg 50 --solve --label $lib >> gpurun_out/ab.txt 2>&1
  done
done
unset RKMF_LIB_PATH
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/ab_gputest.log 2>&1; echo "pytest rc=$?"
