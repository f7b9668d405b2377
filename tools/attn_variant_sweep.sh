for B in 48 96 150 256; do for c in 200 400; do
  for v in default deep team mid; do
    case $v in default) E="";; deep) E="FUSEPLAN_ATTN_DEEP=1";; team) E="FUSEPLAN_ATTN_TEAM=2";; mid) E="FUSEPLAN_ATTN_MID_MAX_B=512";; esac
    r=$(env $E timeout 120 python tools/attn_roofline.py $B $c 2>&1 | tail -1)
    echo "$B $c $v $r"
  done
done; done
