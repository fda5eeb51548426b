D=gpurun_out/ncu; mkdir -p $D
bash tools/ncu_capture.sh k_plane_fwd_cl c5 $D/r2d_c5_plane_fwd_cl
bash tools/ncu_capture.sh k_plane_bwd_cl c5 $D/r2d_c5_plane_bwd_cl
ls -la $D
