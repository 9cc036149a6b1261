"""Executor half of __graft_entry__.smoke() (filled in with the executor)."""


def run_smoke_executor():
    return None
