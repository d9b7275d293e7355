bash tools/variant_run.sh p11 r1 minb3
bash tools/env_variants.sh p11e - MT_CHUNK=256 MT_CHUNK=1024
