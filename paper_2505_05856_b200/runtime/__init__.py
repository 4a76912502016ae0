"""B200 runtime: model graphs, stage executor, 1F1B pipeline, profiler."""
