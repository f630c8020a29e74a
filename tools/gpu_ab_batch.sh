bash tools/gpu_ab.sh r02e NEWTON 6 4 5
bash tools/gpu_ab.sh r02f SPLIT 1 2 4 3
