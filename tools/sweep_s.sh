# E/F L2-prefetch sweep; run on the GPU box
V='[{"engine":"fused-e","PIPECG_B200_BPS":3},{"engine":"fused-e","PIPECG_B200_BPS":3,"PIPECG_B200_L2PF":1},{"engine":"fused-e","PIPECG_B200_BPS":3,"PIPECG_B200_L2PF":2},{"engine":"fused-e","PIPECG_B200_BPS":3,"PIPECG_B200_L2PF":4},{"engine":"fused-f","PIPECG_B200_L2PF":0},{"engine":"fused-f","PIPECG_B200_L2PF":2},{"engine":"fused-f","PIPECG_B200_L2PF":4}]'
timeout 300 python tools/sweep.py 3d7 256 "$V" 2>&1 | tail -7
V2='[{"engine":"fused-f"},{"engine":"fused-f","PIPECG_B200_L2PF":1},{"engine":"fused-f","PIPECG_B200_L2PF":2},{"engine":"fused-f","PIPECG_B200_L2PF":4},{"engine":"fused-e","PIPECG_B200_L2PF":2}]'
timeout 400 python tools/sweep.py 3d27 400 "$V2" 2>&1 | tail -5
