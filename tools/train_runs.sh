# Training experiments (offline; weights into variants/, reports beside them)
set -x
PYTORCH_CUDA_ALLOC_CONF=expandable_segments:True python tools/train3d.py --depth 6 --init random --steps 12000 --lr 1e-3 \
    --n 128 --frames 20 --big 10 --ritz-m 300 --ritz-every 1 --eval256 --seed 61 --out variants/expB12_L6.npm \
    > gpurun_out/r2_trainB12.log 2>&1
cp variants/expB12_L6.* gpurun_out/ 2>/dev/null
