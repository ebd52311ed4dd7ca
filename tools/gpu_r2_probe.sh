set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
cd tools/microbench; ls
for args in "0 256 256 296" "1 256 256 296" "1 256 256 32" "1 256 256 1" "2 256 256 296" "2 256 256 32" "3 256 256 296" "3 256 256 1" "0 512 128 296" "1 512 128 296" "3 512 128 296" "3 512 128 1"; do
  timeout 60 ./reduce $args
done
cd ../..
CONFIGS="0 1 2 3 4" STEPS=5 timeout 900 bash tools/quickbench.sh
