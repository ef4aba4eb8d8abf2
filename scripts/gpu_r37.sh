python scripts/debug_u8_flake.py 40 80 tf32 15 2>&1 | tail -12
python scripts/debug_u8_flake.py 40 80 f16 10 2>&1 | tail -5
python scripts/debug_u8_flake.py 48 64 tf32 10 2>&1 | tail -5
