mkdir -p gpurun_out/train
timeout 1500 python tools/train3d.py --init random --steps 12000 --n 64 --frames 96 --max-sweeps 40 --lr 1e-3 --seed 7 --eval256 --out gpurun_out/train/sc_d.npm > gpurun_out/train/sc_d.log 2>&1; echo d $?; tail -6 gpurun_out/train/sc_d.log
