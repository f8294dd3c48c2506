for e in "X=1" "SGTK_PANEL_FORMAT=2"; do
  p=tf32
  echo "$e $p: $(env $e python tools/agnn_only.py --precision $p | tail -1) dense $(env $e SGTK_PANEL_DEBUG=1 python tools/agnn_only.py --precision $p | tail -1) sparse $(env $e SGTK_PANEL_DEBUG=2 python tools/agnn_only.py --precision $p | tail -1)"
done
python tools/agnn_only.py | head -1
SGTK_PANEL_FORMAT=2 python tools/agnn_only.py | head -1
