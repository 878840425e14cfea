for v in cur lpt0 lpt2 cur lpt0 lpt2; do
  PACKINFER_LIB=$PWD/variants/libpi_$v.so python scripts/shard_sim.py 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$v', ' '.join(f'N{k}: step {v[\"step_ms\"]:.3f} eff {v[\"efficiency_est\"]:.3f} keff {v[\"kernel_eff_est\"]:.3f}' for k,v in d.items()))"
done
