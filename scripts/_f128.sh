bash scripts/gpu_ab.sh cur m3
bash scripts/gpu_geom_variants.sh cur m3 m3x
