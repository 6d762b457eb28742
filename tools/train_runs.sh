# Training experiments (offline; weights into variants/, reports beside them)
set -x
PYTORCH_CUDA_ALLOC_CONF=expandable_segments:True python tools/train3d.py --depth 6 --init random --steps 8000 --lr 1e-3 \
    --n 128 --frames 16 --big 8 --ritz-m 300 --ritz-every 1 --eval256 --seed 51 --out variants/expB10_L6.npm \
    > gpurun_out/r2_trainB10.log 2>&1
cp variants/expB10_L6.* gpurun_out/ 2>/dev/null
PYTORCH_CUDA_ALLOC_CONF=expandable_segments:True python tools/train3d.py --depth 5 --init random --steps 16000 --lr 1e-3 \
    --n 128 --frames 20 --big 10 --ritz-m 300 --ritz-every 1 --eval256 --seed 52 --out variants/expB11_L5.npm \
    > gpurun_out/r2_trainB11.log 2>&1
cp variants/expB11_L5.* gpurun_out/ 2>/dev/null
