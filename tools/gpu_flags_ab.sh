bash tools/exppair.sh c4 base minb2 2
bash tools/exppair.sh c4 base cg 2
bash tools/exppair.sh c4 base minb4 1
