# round-2 auxiliary lines: every config at full length, EPI3 / C4 bench lines, Krylov loop at L9
TAG=${1:-r02c}
mkdir -p gpurun_out
python tools/run_configs.py gpurun_out/configs_$TAG.txt > gpurun_out/configs_$TAG.log 2>&1; echo configs=$?
python tools/kbench.py C4:9 40 3 > gpurun_out/kbench_l9_$TAG.txt 2>&1; echo kb9=$?
python tools/kbench.py C3 40 5 > gpurun_out/kbench_l8_$TAG.txt 2>&1; echo kb8=$?
bash tools/gpu_configs.sh $TAG
