# E/F occupancy sweep with 56-register windowed kernels; run on the GPU box
V='[{"engine":"fused-e","PIPECG_B200_BPS":3},{"engine":"fused-e","PIPECG_B200_BPS":4},{"engine":"fused-f","PIPECG_B200_BPS":2},{"engine":"fused-f","PIPECG_B200_BPS":3},{"engine":"fused-f","PIPECG_B200_BPS":4},{"engine":"fused-e","PIPECG_B200_BPS":3},{"engine":"fused-e","PIPECG_B200_BPS":4}]'
timeout 300 python tools/sweep.py 3d7 256 "$V" 2>&1 | tail -7
V2='[{"engine":"fused-f","PIPECG_B200_BPS":2},{"engine":"fused-f","PIPECG_B200_BPS":3},{"engine":"fused-e","PIPECG_B200_BPS":2},{"engine":"fused-f","PIPECG_B200_BPS":2}]'
timeout 400 python tools/sweep.py 3d27 400 "$V2" 2>&1 | tail -4
timeout 300 python tools/sweep.py 3d7 400 '[{"engine":"fused-e","PIPECG_B200_BPS":3},{"engine":"fused-e","PIPECG_B200_BPS":4}]' 2>&1 | tail -2
