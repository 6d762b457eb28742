# fine-tune the committed model with 128^3 frames and smoother right-hand sides
mkdir -p gpurun_out/train
timeout 1500 python tools/train3d.py --init paper_2310_00177_b200/weights/npsd3d_L4.npm --steps 6000 --n 64 --frames 48 --big 16 --max-sweeps 120 --lr 3e-4 --eval256 --out gpurun_out/train/ft_a.npm > gpurun_out/train/ft_a.log 2>&1; echo a $?; tail -7 gpurun_out/train/ft_a.log
