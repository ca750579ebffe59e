cd $GRAFT_REPO_ROOT
for r in 1 2; do for ca in 0 1 2 3; do for sg in 100; do
  echo "ca=$ca sigma=$sg $(B200TALLY_CLAIM_AHEAD=$ca python tools/short_walk_once.py 10000000 $sg | tail -1)"
done; done; done
