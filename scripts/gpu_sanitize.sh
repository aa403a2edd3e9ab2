#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck on small cases of every kernel family.
out=gpurun_out/${TAG:-sanitize}; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
CASES=("70x37x29 2shoc msd fp64 V" "70x37x29 2shoc dirichlet fp32" "64x33x9 2shoc msd fp64 V" "65x33x9 2shoc msd fp64"
       "40x26x22 2shoc l0 fp64" "40x26x22 cd dirichlet fp32" "70x41 2shoc msd fp64 V" "301 2shoc msd fp64"
       "6001 2shoc msd fp64 V" "6001 cd l0 fp32" "FUSED=1 70x37x29 cd msd fp64 V" "FUSED=1 33x17x9 cd dirichlet fp32"
       "SLABS=3 133x70 2shoc msd fp64 V" "SLABS=3 40x26x22 2shoc msd fp32"
       "ROWS=2 61x11 2shoc msd fp64 V" "ROWS=1 33x5 cd l0 fp32 V" "87x45 2shoc dirichlet fp32" "TILE2D 70x41 2shoc msd fp64 V")
[ -n "$ONLY_NEW" ] && CASES=("${CASES[@]:8}")     # the round-2 kernels only
[ -n "$ONLY_2D" ] && CASES=("70x41 2shoc msd fp64 V" "SLABS=3 133x70 2shoc msd fp64 V" "ROWS=2 61x11 2shoc msd fp64 V" "ROWS=1 33x5 cd l0 fp32 V" "87x45 2shoc dirichlet fp32" "TILE2D 70x41 2shoc msd fp64 V")
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  # 70x37x29: interior (lean), lean edge and ragged tiles; 64x33x9 / 65x33x9: tiles whose ring holds a
  # face point (per-point face path); 40x26x22: all tiles on the lean edge path; 2D: the warp-strip
  # kernel (default; 2- and 1-row chunks, fp32, ragged strips) and the shared-tile kernel
  for c in "${CASES[@]}"; do
    envs=""; args="$c"
    case "$c" in FUSED=1*) envs="NLSE_FUSED=1"; args="${c#FUSED=1 }";; SLABS=*) envs="${c%% *}"; args="${c#* }";;
      ROWS=*) envs="NLSE_STRIP_ROWS=${c%% *}"; envs="NLSE_STRIP_ROWS=${envs#*ROWS=}"; args="${c#* }";;
      TILE2D*) envs="NLSE_2D_KERNEL=tile"; args="${c#TILE2D }";; esac
    env NSTEPS=2 $envs timeout 300 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/debug_case.py $args > $out/${tool}_${c// /_}.log 2>&1
    rc=$?
    echo "$tool [$c] rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|Hazard' $out/${tool}_${c// /_}.log | head -2 | tr '\n' ' ')"
  done
done
