mkdir -p gpurun_out/train
timeout 1200 python tools/train3d.py --init paper_2310_00177_b200/weights/npsd3d_L4.npm --steps 4000 --n 64 --frames 16 --big 16 --max-sweeps 40 --lr 3e-4 --seed 11 --eval256 --out gpurun_out/train/ft_c.npm > gpurun_out/train/ft_c.log 2>&1; echo c $?; tail -6 gpurun_out/train/ft_c.log
timeout 1500 python tools/train3d.py --init random --steps 8000 --n 64 --frames 48 --big 16 --max-sweeps 40 --lr 1e-3 --seed 13 --eval256 --out gpurun_out/train/sc_b.npm > gpurun_out/train/sc_b.log 2>&1; echo b $?; tail -6 gpurun_out/train/sc_b.log
