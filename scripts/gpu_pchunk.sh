PF_PREFIXES=${PF_PREFIXES:-131072} PF_CHUNKS=${PF_CHUNKS:-64,1024,4096} bash scripts/gpu_pf_opt_ab.sh "$@"
