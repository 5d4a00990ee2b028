import cProfile, pstats, sys, os, time
sys.path.insert(0, os.getcwd())
from paper_2212_02224_b200.episodes import run_episodes
from paper_2212_02224_b200.planners import PlannerEnvConfig, make_batch_planner
from paper_2212_02224_b200.sim import RoadSpec, ScenarioConfig
scs = [ScenarioConfig(RoadSpec(4), 1.0, 12, s, episode_length=150) for s in range(256)]
planner = make_batch_planner("mpc-bilevel", PlannerEnvConfig())
run_episodes(scs[:4], planner)
t0 = time.perf_counter(); run_episodes(scs, planner); print("wall", time.perf_counter() - t0)
pr = cProfile.Profile(); pr.enable()
run_episodes(scs, planner)
pr.disable()
st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(14)
