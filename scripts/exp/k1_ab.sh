for i in 1 2; do
python scripts/exp/k1_ab.py --lib r1
python scripts/exp/k1_ab.py --lib new
KLS_TMA_VIRT=148 python scripts/exp/k1_ab.py --lib new
KLS_TMA_VIRT=24 python scripts/exp/k1_ab.py --lib new
KLS_TMA_VIRT=98 python scripts/exp/k1_ab.py --lib new
done
