# Training experiments (offline; weights into variants/, reports beside them)
set -x
PYTORCH_CUDA_ALLOC_CONF=expandable_segments:True python tools/train3d.py --depth 7 --init random --steps 8000 --lr 1e-3 \
    --n 128 --frames 16 --big 8 --ritz-m 300 --ritz-every 1 --eval256 --seed 81 --out variants/expB14_L7.npm \
    > gpurun_out/r2_trainB14.log 2>&1
cp variants/expB14_L7.* gpurun_out/ 2>/dev/null
