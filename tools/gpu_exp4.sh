mkdir -p gpurun_out
VARIANTS="default sm smp p5c6 p5sm p5smp p5c6smp p56 p56smp p56c2" NOPHASES=1 bash tools/vrun.sh 2>&1 | tee gpurun_out/exp4_kbench.log
